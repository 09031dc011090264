# Quick GPU check: GPU tests + one bench line.  usage: bash scripts/gpu_quick.sh <tag>
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_pytest.txt 2>&1
tail -2 gpurun_out/${TAG}_pytest.txt
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.txt 2>&1
python - "$TAG" <<'PY'
import json,sys
for l in open(f"gpurun_out/{sys.argv[1]}_bench.txt"):
    if l.startswith("{"):
        d=json.loads(l); print("frame_ms", d["ms_per_step"], "Mrays/s", d["value"], "stages", d["stages_ms"], "frac", d["roofline"]["frac"], "e2e", d.get("e2e",{}).get("value"), "sweep", {k:(v["ms_per_frame"], v.get("stages_ms")) for k,v in d.get("sweep_ms_per_frame",{}).items()})
PY
