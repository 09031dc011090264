"""Experiment: march kernel time in raster order vs a cost-descending tile
order taken from the previous frame's per-tile evaluation counts."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200 import _capi as capi  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402


def march_ms(rd, cam, c, reps=20):
    out = []
    for i in range(reps + 2):
        rd.profile(True)
        capi.check(rd.lib.bt_trace(rd.ctx, C.byref(cam), C.byref(c), 0, 0, 0), "bt_trace")
        ms, n = rd.profile_read_ex()
        rd.profile(False)
        if i >= 2:
            out.append(ms[5])
    return float(np.median(out))


for name in sys.argv[1:] or ["C1", "C3", "C2", "C5"]:
    s = Scene.build(name)
    rd = Renderer(0)
    rd.upload(s)
    cam, cfg = s.device_camera, RenderConfig()
    c = cfg.to_c()
    rd.render_frame(cam, cfg, exact=False, graph=False)
    g = rd.download_gbuffer()
    H, W = s.height, s.width
    tx, ty = s.tiles
    ev = np.zeros((ty * 8, tx * 8), np.int64)
    ev[:H, :W] = g.evalCount.reshape(H, W)
    t = ev.reshape(ty, 8, tx, 8).transpose(0, 2, 1, 3).reshape(ty * tx, 64)
    capi.check(rd.lib.bt_set_scheduling(rd.ctx, 0), "sched")
    base = march_ms(rd, cam, c)
    res = {"raster": base}
    capi.check(rd.lib.bt_set_scheduling(rd.ctx, 1), "sched")
    res["lpt(device)"] = march_ms(rd, cam, c)
    for key, cost in (("sum", t.sum(1)), ("max", t.max(1)), ("sum+max", t.sum(1) / 32 + t.max(1))):
        order = np.argsort(-cost, kind="stable").astype(np.uint32)
        capi.check(rd.lib.bt_set_tile_order(rd.ctx, order.ctypes.data_as(C.c_void_p), len(order)), "order")
        res[key] = march_ms(rd, cam, c)
        g2 = rd.download_gbuffer()
        assert g2.depth.tobytes() == g.depth.tobytes() and g2.evalCount.tobytes() == g.evalCount.tobytes()
    capi.check(rd.lib.bt_set_scheduling(rd.ctx, 1), "sched")
    print(name, {k: round(v, 4) for k, v in res.items()})
    rd.close()
