"""Same-frame cost proxies for longest-first scheduling (available before the
march) vs the measured per-tile cost: march ms under each order."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200 import _capi as capi  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402


def march_ms(rd, cam, c, reps=15):
    out = []
    for i in range(reps + 2):
        rd.profile(True)
        capi.check(rd.lib.bt_trace(rd.ctx, C.byref(cam), C.byref(c), 0, 0, 0), "bt_trace")
        ms, n = rd.profile_read_ex()
        rd.profile(False)
        if i >= 2:
            out.append(ms[5])
    return float(np.median(out))


for name in sys.argv[1:] or ["C3", "C5", "C2", "C1"]:
    s = Scene.build(name)
    rd = Renderer(0)
    rd.upload(s)
    cam, cfg = s.device_camera, RenderConfig()
    c = cfg.to_c()
    rd.lib.bt_set_scheduling(rd.ctx, 0)
    rd.render_frame(cam, cfg, exact=False, graph=False)
    g = rd.download_gbuffer()
    off, fr = rd.download_abuffer()
    H, W = s.height, s.width
    tx, ty = s.tiles
    ev = np.zeros((ty * 8, tx * 8), np.int64)
    ev[:H, :W] = g.evalCount.reshape(H, W)
    t = ev.reshape(ty, 8, tx, 8).transpose(0, 2, 1, 3).reshape(ty * tx, 64)
    cnt = np.diff(off.astype(np.int64))
    tid = np.repeat(np.arange(len(cnt)), cnt)
    span = np.zeros(len(cnt))
    np.add.at(span, tid, (fr["zExit"] - fr["zEntry"]).astype(np.float64))
    spanmax = np.zeros(len(cnt))
    np.maximum.at(spanmax, tid, (fr["zExit"] - fr["zEntry"]).astype(np.float64))
    # view-z extents (linear in depth, like the march steps)
    cam14 = cam
    inv_near, idr = cam.invNear, cam.invDepthRange
    vz = lambda z: 1.0 / (inv_near - z / idr)  # noqa: E731  (view_z_from_ndc)
    vspan = np.zeros(len(cnt))
    np.add.at(vspan, tid, (vz(fr["zExit"].astype(np.float64)) - vz(fr["zEntry"].astype(np.float64))))
    vmax = np.zeros(len(cnt))
    np.maximum.at(vmax, tid, (vz(fr["zExit"].astype(np.float64)) - vz(fr["zEntry"].astype(np.float64))))
    res = {"raster": march_ms(rd, cam, c)}
    for key, cost in (("truth:max", t.max(1)), ("cnt", cnt), ("span", span), ("vspan", vspan), ("vmax", vmax),
                      ("cnt+4span", 4 * cnt + 16 * span), ("vspan+cnt", vspan / max(vspan.mean(), 1e-9) + cnt / max(cnt.mean(), 1e-9))):
        order = np.argsort(-cost, kind="stable").astype(np.uint32)
        capi.check(rd.lib.bt_set_tile_order(rd.ctx, order.ctypes.data_as(C.c_void_p), len(order)), "order")
        res[key] = march_ms(rd, cam, c)
        r = np.corrcoef(cost[cnt > 0], t.max(1)[cnt > 0])[0, 1]
        res[key + " r"] = r
    print(name, {k: round(v, 3) for k, v in res.items()})
    rd.close()
