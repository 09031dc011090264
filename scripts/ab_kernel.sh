# A/B of kernels' device time across library variants (lib/ab/lib<V>.so from
# scripts/build_variant.sh): ncu launch list (cold-cache, serialised) per
# variant and config, mean us per launch of the kernels matching $KERN (a
# regex), skipping the first two launches.  FRAMES=1 profiles whole bench
# frames (bench.py) instead of march_bench.py's stage-(c) repeats.
#   usage: VARS="A B" CFGS="C3 C5" KERN="k_view_build|k_march" bash scripts/ab_kernel.sh
LIB=paper_2304_09673_b200/lib/libblobtree_b200.so
cp $LIB /tmp/lib_current.so
mkdir -p gpurun_out
for v in ${VARS:-A B}; do
  cp paper_2304_09673_b200/lib/ab/lib$v.so $LIB
  for cfg in ${CFGS:-C3 C5}; do
    if [ -n "$FRAMES" ]; then CMD="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-sweep"
    else CMD="python scripts/march_bench.py $cfg 3"; fi
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:${KERN:-k_march}" -c ${NLAUNCH:-12} --csv \
      --log-file gpurun_out/ab_${v}_${cfg}.csv $CMD > /dev/null 2>&1
    python - "$v" "$cfg" gpurun_out/ab_${v}_${cfg}.csv <<'PY'
import csv, sys, collections
agg = collections.defaultdict(list)
for d in csv.DictReader(l for l in open(sys.argv[3]) if not l.startswith("==")):
    s = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}[d["Metric Unit"]]
    agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")) * s)
for k, v in agg.items():
    print(sys.argv[1], sys.argv[2], k[-40:], f"{sum(v[2:]) / max(1, len(v[2:])):.1f} us  (n={len(v)})")
PY
  done
done
cp /tmp/lib_current.so $LIB
