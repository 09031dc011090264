# Per-kernel launch list (ncu, cold, serialised) for a config.  usage: bash scripts/gpu_launches.sh <tag> <config>
TAG=${1:-l}; CFG=${2:-C3}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_ncu1.txt 2>&1
