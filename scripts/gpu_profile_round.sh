# Round profiles: per config a bench line, the ncu launch list, and --set full captures
# (+ the FP32 instruction counters of SURVEY 8(d)) of the named kernels.
#   usage: bash scripts/gpu_profile_round.sh <tag-prefix> "<CFG>:<k1,k2>" ["<CFG>:<k1>" ...]
#   e.g.   bash scripts/gpu_profile_round.sh r02p "C3:k_march,k_tile_raster,k_tile_views" "C5:k_march,k_view_build"
P=$1; shift
mkdir -p gpurun_out
FP=smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum
for spec in "$@"; do
  CFG=${spec%%:*}; KS=${spec#*:}; TAG=${P}$(echo $CFG | tr 'A-Z' 'a-z')
  timeout 400 python bench.py --config $CFG --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_bench.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
     python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_ncu1.txt 2>&1
  for K in $(echo $KS | tr ',' ' '); do
    timeout 600 ncu --set full --metrics $FP --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
       -o gpurun_out/${TAG}_prof_$K python bench.py --config $CFG --steps 1 --warmup 2 --no-cpu-baseline --no-sweep \
       > gpurun_out/${TAG}_ncu_$K.txt 2>&1
  done
  ls gpurun_out | grep "^${TAG}_" | tr '\n' ' '; echo
done
