"""Experiment: two contexts, each rendering half of the tile rows on its own
stream, launched back to back (graph replays) -- does the GPU overlap one
half's A-buffer / views with the other half's march?"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
s = Scene.build(name)
cfg = RenderConfig()
cam = s.device_camera
tx, ty = s.tiles
dev = torch.device("cuda", 0)


def timeit(fn, reps=50):
    import time
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


# one context, full frame
st0 = torch.cuda.Stream(dev)
r0 = Renderer(0)
r0.set_stream(st0.cuda_stream)
r0.upload(s)
full = timeit(lambda: r0.render_frame(cam, cfg, exact=False, graph=True))
# two contexts, half frames on two streams
for parts in (2, 3, 4):
    rows = np.linspace(0, ty, parts + 1).round().astype(int)
    rs = []
    for k in range(parts):
        st = torch.cuda.Stream(dev)
        r = Renderer(0)
        r.set_stream(st.cuda_stream)
        r.upload(s)
        rs.append((r, int(rows[k] * tx), int(rows[k + 1] * tx)))

    def both():
        for r, t0, t1 in rs:
            r.render_frame(cam, cfg, exact=False, graph=True, tile0=t0, tile1=t1, normals=False)

    split = timeit(both)
    print(name, f"full frame {full:.4f} ms, {parts} concurrent tile-row parts (no normals) {split:.4f} ms")
