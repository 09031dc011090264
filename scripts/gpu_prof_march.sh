# ncu --set full captures of k_march (plus the FP32 instruction counters SURVEY 8(d) names) for
# each config given.  usage: bash scripts/gpu_prof_march.sh <tag> C3 [C5 ...]
TAG=$1; shift
mkdir -p gpurun_out
FP=smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum
for CFG in "$@"; do
  timeout 600 ncu --set full --metrics $FP --clock-control none --import-source on -k regex:k_march -s 2 -c 1 \
     -o gpurun_out/${TAG}_${CFG}_prof_k_march python bench.py --config $CFG --steps 1 --warmup 2 --no-cpu-baseline --no-sweep \
     > gpurun_out/${TAG}_${CFG}_ncu.txt 2>&1
  tail -2 gpurun_out/${TAG}_${CFG}_ncu.txt
done
ls gpurun_out | grep ${TAG}_
