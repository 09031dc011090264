"""Experiment: frames in flight.  Two contexts (each with its own tree copy,
buffers, CUDA graph and stream) render alternate frames of the perturbed
sequence, so one frame's latency-bound stages (A-buffer, view compilation,
normals) can run while the other frame's march fills the GPU.  Compares the
per-frame throughput with one context rendering the same frames back to back.
usage: python scripts/inflight_exp.py [CONFIG] [FRAMES]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40
s = Scene.build(name)
cfg, cam = RenderConfig(), s.device_camera
dev = torch.device("cuda", 0)
perturbed = s.name in ("C3", "C4")
deltas = []
if perturbed:
    for f in range(8):
        w, p, c = s.perturb(f)
        deltas.append((torch.from_numpy(w.view(np.int32)).to(dev), torch.from_numpy(p).to(dev),
                       torch.from_numpy(c.view(np.int32)).to(dev)))


def make(n):
    out = []
    for _ in range(n):
        st = torch.cuda.Stream(dev)
        r = Renderer(0)
        r.set_stream(st.cuda_stream)
        r.upload(s)
        out.append((r, st))
    return out


def run(ctxs, k):
    for i in range(k):
        r, _ = ctxs[i % len(ctxs)]
        if perturbed:
            w, p, c = deltas[i % len(deltas)]
            r.update_params_device(w.data_ptr(), p.data_ptr(), c.data_ptr(), len(s.prims))
        r.render_frame(cam, cfg, exact=False, graph=True)


for n in (1, 2, 3):
    ctxs = make(n)
    run(ctxs, 2 * n)  # capture the graphs
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(ctxs, frames)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / frames
    print(f"{name}: {n} context(s) in flight: {dt * 1e3:.4f} ms/frame, {s.width * s.height / dt / 1e6:.0f} Mrays/s")
    for r, _ in ctxs:
        r.close()
