# Multi-rank checks on ONE GPU (IPC fused gather + per-rank normals): the fused-gather
# tests at 2 and 3 ranks and the bench's multi-rank path at 2 ranks.  usage: bash scripts/gpu_multi.sh <tag>
TAG=${1:-m}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_gather.py -q -m gpu -x > gpurun_out/${TAG}_fused.txt 2>&1
tail -3 gpurun_out/${TAG}_fused.txt
BT_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench2.txt 2>&1
grep '^{' gpurun_out/${TAG}_bench2.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('value','ms_per_step','e2e','scaling_c4')})"
tail -3 gpurun_out/${TAG}_bench2.txt | grep -v '^{'
