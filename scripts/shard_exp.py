"""Per-rank work of an N-way tile-row split, measured on one GPU: graph
replays of render_frame over each rank's rows (no normals, no gather).
The max over ranks is the critical path of the sharded frame."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200.distributed import tile_row_ranges  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
s = Scene.build(name)
cfg, cam = RenderConfig(), s.device_camera
tx, ty = s.tiles
st = torch.cuda.Stream()
rd = Renderer(0)
rd.set_stream(st.cuda_stream)
rd.upload(s)


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


full = timed(lambda: rd.render_frame(cam, cfg, exact=False, graph=True))
print(name, f"full frame {full:.4f} ms")
for n in (2, 4, 8):
    rows = tile_row_ranges(ty, n)
    per = []
    for r in range(n):
        t0, t1 = int(rows[r] * tx), int(rows[r + 1] * tx)
        per.append(timed(lambda: rd.render_frame(cam, cfg, exact=False, graph=True, tile0=t0, tile1=t1,
                                                  normals=False)))
    print(name, n, "ranks: per-rank ms", np.round(per, 4), f"max {max(per):.4f} -> ideal speed-up {full / max(per):.2f}")

# cost-balanced split: per-row cost = the full frame's evaluation count of the
# row (what the bench's multi-GPU path measures in its warm-up frames)
rd.render_frame(cam, cfg, exact=False, graph=False)
g = rd.download_gbuffer()
ev = np.zeros((ty * 8, tx * 8), np.float64)
ev[:s.height, :s.width] = g.evalCount.reshape(s.height, s.width)
row_cost = ev.reshape(ty, 8, tx * 8).sum(axis=(1, 2))
for n in (2, 4, 8):
    for label, cost in (("evals", row_cost), ("evals+tiles", row_cost + row_cost.sum() / ty * 0.25)):
        rows = tile_row_ranges(ty, n, cost)
        per = []
        for r in range(n):
            t0, t1 = int(rows[r] * tx), int(rows[r + 1] * tx)
            per.append(timed(lambda: rd.render_frame(cam, cfg, exact=False, graph=True, tile0=t0, tile1=t1,
                                                      normals=False)))
        print(name, n, f"ranks balanced by {label}: per-rank ms", np.round(per, 4),
              f"max {max(per):.4f} -> ideal speed-up {full / max(per):.2f}")

# stage split of one middle rank at 8-way (eager frames, CUDA-event profile)
import ctypes as C  # noqa: E402
from paper_2304_09673_b200 import _capi as capi  # noqa: E402
rows = tile_row_ranges(ty, 8)
t0, t1 = int(rows[3] * tx), int(rows[4] * tx)
rd.profile(True)
lib, c = rd.lib, cfg.to_c()
for _ in range(5):
    capi.check(lib.bt_roi(rd.ctx, None, 0), "roi")
    capi.check(lib.bt_voi_build(rd.ctx, C.c_float(cfg.hitEpsilon)), "voi")
    capi.check(lib.bt_abuffer_build(rd.ctx, C.byref(cam), t0, t1), "ab")
    capi.check(lib.bt_trace(rd.ctx, C.byref(cam), C.byref(c), t0, t1, 0), "trace")
ms, n = rd.profile_read_ex()
print(name, "rank 3/8 stage ms [roi_voi, abuffer, trace, normals, views, march]:", np.round(ms / np.maximum(n, 1), 4))
