"""Depth slabs (bt_set_depth_slabs): frame time and A-buffer footprint per
slab count.  For n slabs the frame's A-buffer is built n times, each time for
one slab's camera (the slab_camera rule of capi.cu: view depth [near, far]
in n equal parts); the peak fragment count over the slabs is what the
A-buffer must hold, against the single pass's total.

    python scripts/depth_slabs.py [C3 C4 ...]
"""
import copy
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200 import _capi as capi  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402


def slab_camera(cam, s, n):
    k = copy.copy(cam)
    rng = cam.farZ - cam.nearZ
    k.nearZ = cam.nearZ if s == 0 else cam.nearZ + rng * s / n
    k.farZ = cam.farZ if s == n - 1 else cam.nearZ + rng * (s + 1) / n
    k.invNear = 1.0 / k.nearZ
    k.invDepthRange = 1.0 / (k.invNear - 1.0 / k.farZ)
    return k


for name in sys.argv[1:] or ["C3", "C4"]:
    s = Scene.build(name)
    rd = Renderer(0)
    rd.upload(s)
    cam = s.device_camera
    cfg = RenderConfig()
    for n in (1, 2, 4, 8):
        rd.set_depth_slabs(n)
        peak = 0
        for k in range(n):
            rd.render_frame(cam, cfg, exact=False, graph=False)  # VOIs of the frame
            _, frags = rd.rasterize_volumes(slab_camera(cam, k, n))
            peak = max(peak, len(frags))
        for _ in range(3):
            rd.render_frame(cam, cfg, exact=False, graph=True)
        capi.check(rd.lib.bt_sync(rd.ctx), "bt_sync")
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            rd.render_frame(cam, cfg, exact=False, graph=True)
        capi.check(rd.lib.bt_sync(rd.ctx), "bt_sync")
        ms = (time.perf_counter() - t0) * 1e3 / reps
        st = rd.stats()
        print(f"{name} slabs {n}: {ms:.3f} ms/frame (graph replays, wall clock), peak fragments per slab {peak}, "
              f"field evals {st.fieldEvals}")
    rd.close()
