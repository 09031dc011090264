"""March time over a perturbed frame sequence (C3 bench workload) under
different tile orders, eager frames with CUDA-event profiling."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
s = Scene.build(name)
frames = [s.perturb(f) for f in range(16)]
tx, ty = s.tiles
H, W = s.height, s.width


def tile_cost(g, dil):
    ev = np.zeros((ty * 8, tx * 8), np.int64)
    ev[:H, :W] = g.evalCount.reshape(H, W)
    t = ev.reshape(ty, 8, tx, 8).max(axis=(1, 3))
    for _ in range(dil):
        p = np.pad(t, 1)
        t = np.max([p[1 + dy:1 + dy + ty, 1 + dx:1 + dx + tx] for dy in (-1, 0, 1) for dx in (-1, 0, 1)], axis=0)
    return t.reshape(-1)


for mode in ("raster", "device", "prev", "prev-dil1", "prev-dil2", "same"):
    rd = Renderer(0)
    rd.upload(s)
    cam, cfg = s.device_camera, RenderConfig()
    rd.lib.bt_set_scheduling(rd.ctx, 1 if mode == "device" else 0)
    ms = []
    prev = None
    for f, (w, p, c) in enumerate(frames):
        rd.update_params(w, p, c)
        if mode == "same":  # oracle: this frame's own costs (needs a first pass)
            rd.render_frame(cam, cfg, exact=False, graph=False)
            prev = rd.download_gbuffer()
        if prev is not None and mode not in ("raster", "device"):
            dil = 1 if mode == "prev-dil1" else 2 if mode == "prev-dil2" else 0
            order = np.argsort(-tile_cost(prev, dil), kind="stable").astype(np.uint32)
            assert rd.lib.bt_set_tile_order(rd.ctx, order.ctypes.data_as(C.c_void_p), len(order)) == 0
        rd.profile(True)
        rd.render_frame(cam, cfg, exact=False, graph=False)
        m, n = rd.profile_read_ex()
        rd.profile(False)
        prev = rd.download_gbuffer()
        if f >= 3:
            ms.append(m[5] / max(1, n[5]))
    print(name, mode, "march ms median", round(float(np.median(ms)), 4))
    rd.close()
