# One GPU round: tests, smoke, bench, launch list, full ncu captures of the top kernels.
# usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${TAG}_nvsmi.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_bench.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_ncu1.txt 2>&1
for K in k_march k_raster k_view_count k_view_fetch; do
  timeout 500 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/${TAG}_prof_$K python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-sweep > gpurun_out/${TAG}_ncu_$K.txt 2>&1
done
tail -3 gpurun_out/${TAG}_pytest.txt; tail -2 gpurun_out/${TAG}_smoke.txt; tail -c 3000 gpurun_out/${TAG}_bench.txt
