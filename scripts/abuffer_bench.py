"""Stable timing of stage (b) alone: N repeated bt_abuffer_build calls
(camera products reused) with CUDA-event profiling; prints the median.
    python scripts/abuffer_bench.py [C3] [reps]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200 import _capi as capi  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
s = Scene.build(name)
rd = Renderer(0)
rd.upload(s)
cam = s.device_camera
cfg = RenderConfig()
rd.render_frame(cam, cfg, exact=False, graph=False)
lib = rd.lib
ab = []
for i in range(reps + 3):
    rd.profile(True)
    capi.check(lib.bt_abuffer_build(rd.ctx, C.byref(cam), 0, 0), "bt_abuffer_build")
    ms, n = rd.profile_read_ex()
    rd.profile(False)
    if i >= 3:
        ab.append(ms[1])
print(f"{name} abuffer_ms {np.median(ab):.4f} min {min(ab):.4f}")
