# ncu launch list (per-kernel device time, cold-cache, serialised) of the bench frame for each config.
#   usage: bash scripts/gpu_launches_cfg.sh <tag> C3 [C4 ...]
TAG=$1; shift
mkdir -p gpurun_out
for CFG in "$@"; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_${CFG}_launches.csv \
     python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_${CFG}_ncu1.txt 2>&1
done
python scripts/launch_table.py gpurun_out/${TAG}_*_launches.csv
