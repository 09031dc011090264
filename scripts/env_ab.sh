# whole-frame A/B of environment switches on one build: bench.py ms_per_step, alternating.
#   ENVS="BT_RAY_ORDER=0 BT_RAY_ORDER=1" CFGS="C3 C5" bash scripts/env_ab.sh
for r in 1 2 3; do
  for e in ${ENVS}; do
    for cfg in ${CFGS:-C3}; do
      echo "$e $cfg $(env $e timeout 200 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-sweep 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
    done
  done
done
