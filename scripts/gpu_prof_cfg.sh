# Full ncu capture of one kernel for a config.  usage: bash scripts/gpu_prof_cfg.sh <tag> <config> <kernel-regex>
TAG=$1; CFG=$2; K=$3
mkdir -p gpurun_out
timeout 500 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/${TAG}_prof_$K python bench.py --config $CFG --steps 1 --warmup 2 --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_ncu_$K.txt 2>&1
