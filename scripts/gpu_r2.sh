# Round-2 GPU check: the new reference-scale parity tests, the whole GPU suite, one bench line.
#   usage: bash scripts/gpu_r2.sh <tag> [pytest -k expr]
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_reference_scale.py -q -s -m gpu ${2:+-k "$2"} > gpurun_out/${TAG}_scale.txt 2>&1
tail -5 gpurun_out/${TAG}_scale.txt
timeout 900 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_reference_scale.py > gpurun_out/${TAG}_pytest.txt 2>&1
tail -2 gpurun_out/${TAG}_pytest.txt
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.txt 2>&1
python - "$TAG" <<'PY'
import json,sys
for l in open(f"gpurun_out/{sys.argv[1]}_bench.txt"):
    if l.startswith("{"):
        d=json.loads(l); print("frame_ms", d["ms_per_step"], "Mrays/s", d["value"], "stages", d["stages_ms"], "frac", d["roofline"]["frac"], "e2e", d.get("e2e",{}).get("value"), "sweep", {k:(v["ms_per_frame"], v.get("stages_ms")) for k,v in d.get("sweep_ms_per_frame",{}).items()})
PY
tail -3 gpurun_out/${TAG}_bench.txt | grep -v '^{'
