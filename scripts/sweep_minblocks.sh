# Sweep the k_trace register budget (blocks/SM the compiler must fit).
mkdir -p gpurun_out
for mb in 8 6 5 4; do
  BT_TRACE_MINBLOCKS=$mb timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/sweep_mb$mb.txt 2>&1
  python - "$mb" <<'PY'
import json,sys
mb=sys.argv[1]
for l in open(f"gpurun_out/sweep_mb{mb}.txt"):
    if l.startswith("{"):
        d=json.loads(l); print("minblocks", mb, "frame_ms", d["ms_per_step"], "trace_ms", d["stages_ms"]["trace"], "march_ms", d["stages_ms"]["trace_march"], "util", d["frame_stats"]["laneUtilisation"], "frac", d["roofline"]["frac"])
PY
done
