"""Stable timing of stage (c) alone: one frame's A-buffer, then N repeated
bt_trace calls with CUDA-event profiling; prints median views / march ms and
the march kernel's FP32 fraction.  usage: python scripts/march_bench.py [C3] [reps]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200 import _capi as capi  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
exact = "--exact" in sys.argv
s = Scene.build(name)
rd = Renderer(0)
rd.upload(s)
cam = s.device_camera
cfg = RenderConfig()
rd.render_frame(cam, cfg, exact=exact, graph=False)
lib, c = rd.lib, cfg.to_c()
views, march = [], []
for i in range(reps + 3):
    rd.reset_stats()
    rd.profile(True)
    capi.check(lib.bt_trace(rd.ctx, C.byref(cam), C.byref(c), 0, 0, int(exact)), "bt_trace")
    ms, n = rd.profile_read_ex()
    rd.profile(False)
    if i >= 3:
        views.append(ms[4])
        march.append(ms[5])
st = rd.stats()
peak = C.c_float()
capi.check(lib.bt_fp32_peak(0, C.byref(peak), None), "bt_fp32_peak")
m = float(np.median(march))
print(f"{name} views_ms {np.median(views):.4f} march_ms {m:.4f} (min {min(march):.4f}) "
      f"frac {st.fieldFlops / (m * 1e-3) / 1e12 / peak.value:.4f} evals {st.fieldEvals} steps {st.warpSteps} "
      f"util {st.fieldEvals / max(1, 32 * st.warpSteps):.4f} nodes/eval {st.retainedNodeVisits / max(1, st.fieldEvals):.2f} "
      f"flops/eval {st.fieldFlops / max(1, st.fieldEvals):.1f} maxOverlap {st.maxOverlap}")
