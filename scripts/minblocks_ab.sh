# Alternating march-only timing over register budgets (BT_TRACE_MINBLOCKS).
for round in 1 2 3; do
  for mb in ${MBS:-5 6 7}; do
    for cfg in C3 C5; do echo "M$mb $cfg $(BT_TRACE_MINBLOCKS=$mb timeout 100 python scripts/march_bench.py $cfg 30 2>&1 | tail -1 | awk '{print $5}')"; done
  done
done
