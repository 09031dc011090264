# A/B timing of two builds of the library (paper_2304_09673_b200/lib/ab/libA.so
# and libB.so), alternated to cancel box drift: march-only ms per config.
LIB=paper_2304_09673_b200/lib/libblobtree_b200.so
cp $LIB /tmp/lib_current.so
for round in 1 2 3; do
  for v in A B; do
    cp paper_2304_09673_b200/lib/ab/lib$v.so $LIB
    for cfg in ${CFGS:-C3 C5 C1}; do
      echo "$v $cfg $(timeout 100 python scripts/march_bench.py $cfg 40 2>&1 | tail -1 | awk '{print $3, $5}')"
    done
  done
done
cp /tmp/lib_current.so $LIB
