# Experiment: march-only time under cost-proxy variants: add `#if BT_PROXY == k` branches
# around the tileCost formula in k_view_count, then PV="0 1 .." bash scripts/proxy_ab.sh
for pv in ${PV:-0}; do
  make -B lib NVCC="nvcc -DBT_PROXY=$pv" > gpurun_out/proxy_build_$pv.txt 2>&1 || { tail -3 gpurun_out/proxy_build_$pv.txt; continue; }
  cp paper_2304_09673_b200/lib/libblobtree_b200.so /tmp/libP$pv.so
done
LIB=paper_2304_09673_b200/lib/libblobtree_b200.so
for round in 1 2 3; do
  for pv in ${PV:-0 1 2 3}; do
    cp /tmp/libP$pv.so $LIB
    for cfg in C3 C5 C1; do echo "P$pv $cfg $(timeout 100 python scripts/march_bench.py $cfg 30 2>&1 | tail -1 | awk '{print $5}')"; done
  done
done
make -B lib > /dev/null 2>&1
