for b in 0.35 0.7; do for cfg in C3 C5 C1; do echo "B$b $cfg $(BT_SPLIT_BETA=$b timeout 100 python scripts/march_bench.py $cfg 30 2>&1 | tail -1 | awk '{print $5}')"; done; done
