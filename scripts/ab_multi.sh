# A/B/... timing of library variants (paper_2304_09673_b200/lib/ab/lib<V>.so, built by
# scripts/build_variant.sh), alternated over rounds to cancel box drift; march-only ms.
#   usage: VARS="A B C" CFGS="C3 C5" bash scripts/ab_multi.sh
LIB=paper_2304_09673_b200/lib/libblobtree_b200.so
cp $LIB /tmp/lib_current.so
for round in 1 2 3; do
  for v in ${VARS:-A B}; do
    cp paper_2304_09673_b200/lib/ab/lib$v.so $LIB
    for cfg in ${CFGS:-C3 C5 C1}; do
      echo "$v $cfg $(timeout 100 python ${BENCH:-scripts/march_bench.py} $cfg 40 2>&1 | tail -1)"
    done
  done
done
cp /tmp/lib_current.so $LIB
