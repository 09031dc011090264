# Experiment: register budget of the view kernels (BT_VIEW_MINB blocks/SM), alternating A/B.
for mb in ${VMB:-1 8}; do
  make -B lib NVCC="nvcc -DBT_VIEW_MINB=$mb" > gpurun_out/vmb_build_$mb.txt 2>&1 && cp paper_2304_09673_b200/lib/libblobtree_b200.so /tmp/libV$mb.so
done
LIB=paper_2304_09673_b200/lib/libblobtree_b200.so
for round in 1 2 3; do for mb in ${VMB:-1 8}; do cp /tmp/libV$mb.so $LIB
  for cfg in C3 C5; do echo "V$mb $cfg $(timeout 100 python scripts/march_bench.py $cfg 30 2>&1 | tail -1 | awk '{print $3}')"; done
done; done
make -B lib > /dev/null 2>&1
