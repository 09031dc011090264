# Sweep the half-tile split rule (beta x average work per warp).
for b in 1000 2 1 0.5 0.25 0.1; do
  for c in C3 C1 C2 C5; do BT_SPLIT_BETA=$b python scripts/march_bench.py $c 15 | sed "s/^/beta=$b /"; done
done
