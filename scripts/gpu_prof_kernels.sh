# ncu --set full captures of named kernels for a config.  usage: bash scripts/gpu_prof_kernels.sh <tag> <cfg> <regex> [<regex> ...]
TAG=$1; CFG=$2; shift 2
mkdir -p gpurun_out
for K in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
     -o gpurun_out/${TAG}_${CFG}_prof_$K python bench.py --config $CFG --steps 1 --warmup 2 --no-cpu-baseline --no-sweep \
     > gpurun_out/${TAG}_${CFG}_ncu_$K.txt 2>&1
  tail -1 gpurun_out/${TAG}_${CFG}_ncu_$K.txt
done
