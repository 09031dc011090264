# whole-frame A/B of library variants: bench.py ms_per_step, alternating
LIB=paper_2304_09673_b200/lib/libblobtree_b200.so
cp $LIB /tmp/lib_current.so
for r in 1 2 3; do
  for v in ${VARS}; do
    cp paper_2304_09673_b200/lib/ab/lib$v.so $LIB
    for cfg in ${CFGS:-C3}; do
      echo "$v $cfg $(timeout 200 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-sweep 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
    done
  done
done
cp /tmp/lib_current.so $LIB
