# Experiment: register budget of k_raster / k_camera (BT_RASTER_MINB CTAs per SM), alternating.
for mb in ${RMB:-1 4}; do
  make -B lib NVCC="nvcc -DBT_RASTER_MINB=$mb" > gpurun_out/rmb_build_$mb.txt 2>&1 && cp paper_2304_09673_b200/lib/libblobtree_b200.so /tmp/libR$mb.so
done
LIB=paper_2304_09673_b200/lib/libblobtree_b200.so
for round in 1 2; do for mb in ${RMB:-1 4}; do cp /tmp/libR$mb.so $LIB
  python bench.py --no-cpu-baseline --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R$mb', d['stages_ms']['abuffer'], d['ms_per_step'])"
done; done
make -B lib > /dev/null 2>&1
