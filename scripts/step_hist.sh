# Experiment: histogram of active lanes per k_march lockstep step (rebuilds
# with -DBT_STEP_HIST, prints the last launch's histogram per config).
make -B lib NVCC="nvcc -DBT_STEP_HIST" > gpurun_out/stephist_build.txt 2>&1 || { tail -5 gpurun_out/stephist_build.txt; exit 1; }
for cfg in ${CFGS:-C1 C3 C5}; do
  echo "$cfg $(python scripts/march_bench.py $cfg 3 2>&1 | grep STEPHIST | tail -1)"
done
make -B lib > /dev/null 2>&1
