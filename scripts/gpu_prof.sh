# Launch list + full ncu captures of the named kernels.  usage: bash scripts/gpu_prof.sh <tag> <regex1> [<regex2> ...]
TAG=${1:-p}; shift
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_ncu1.txt 2>&1
for K in "$@"; do
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/${TAG}_prof_$K python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_ncu_$K.txt 2>&1
done
ls gpurun_out | grep ${TAG}_
