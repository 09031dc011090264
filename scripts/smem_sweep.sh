# Sweep the march kernel's shared-memory parameter-block capacity
# (BT_MARCH_BLOCKS, float4s per warp; views with more blocks take the
# raw-parameter path) against its register budget (BT_TRACE_MINBLOCKS):
# fewer blocks per warp lets more CTAs fit per SM.  Rebuilds the library.
mkdir -p gpurun_out
for mbk in ${MBK:-320 192 128}; do
  make -B lib NVCC="nvcc -DBT_MARCH_BLOCKS=$mbk" > gpurun_out/smem_build_$mbk.txt 2>&1 || { tail -5 gpurun_out/smem_build_$mbk.txt; continue; }
  for mb in ${MB:-6 7 8}; do
    for cfg in ${CFGS:-C3 C5}; do
      echo "blocks=$mbk minblocks=$mb $(BT_TRACE_MINBLOCKS=$mb timeout 200 python scripts/march_bench.py $cfg 30 2>&1 | tail -1)"
    done
  done
done
make -B lib > /dev/null 2>&1
