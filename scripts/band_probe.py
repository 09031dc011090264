"""Feasibility probe: one frame rendered as K tile-row bands by K contexts on
K streams of ONE GPU (each band's latency-bound prefix overlapping the other
bands' marches).  Each context writes its own G-buffer here (no normals
halo exchange), so this bounds what intra-frame banding can gain.

    python scripts/band_probe.py [C3] [K ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200.distributed import row_costs, tile_row_ranges  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
Ks = [int(k) for k in sys.argv[2:]] or [1, 2, 3, 4]
dev = torch.device("cuda", 0)
cfg = RenderConfig()
base = Scene.build(name)
tiles_x, tiles_y = base.tiles
rd0 = Renderer(0)
rd0.upload(base)
rd0.render_frame(base.device_camera, cfg, exact=False, graph=False)
costs = row_costs(rd0.download_gbuffer().evalCount, base.width, base.height)
rd0.close()
frames = 30
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for K in Ks:
    rows = tile_row_ranges(tiles_y, K, costs)
    streams = [torch.cuda.Stream(dev) for _ in range(K)]
    ctxs, scenes, deltas = [], [], []
    for k in range(K):
        s = Scene.build(name)
        rd = Renderer(0)
        rd.set_stream(streams[k].cuda_stream)
        rd.upload(s)
        ctxs.append(rd)
        scenes.append(s)
        fr = [s.perturb(f) for f in range(frames)]
        deltas.append([(torch.from_numpy(w.view(np.int32)).to(dev), torch.from_numpy(p).to(dev),
                        torch.from_numpy(c.view(np.int32)).to(dev)) for w, p, c in fr])
    t0s = [int(rows[k] * tiles_x) for k in range(K)]
    t1s = [int(rows[k + 1] * tiles_x) for k in range(K)]
    if K == 1:
        t0s, t1s = [0], [0]
    main = torch.cuda.current_stream(dev)

    def frame(f):
        start = torch.cuda.Event()
        start.record(main)
        done = []
        for k in range(K):
            streams[k].wait_event(start)
            w, p, c = deltas[k][f]
            ctxs[k].update_params_device(w.data_ptr(), p.data_ptr(), c.data_ptr(), len(scenes[k].prims))
            ctxs[k].render_frame(scenes[k].device_camera, cfg, exact=False, graph=True, tile0=t0s[k], tile1=t1s[k],
                                 normals=True)
            e = torch.cuda.Event()
            e.record(streams[k])
            done.append(e)
        for e in done:
            main.wait_event(e)

    for f in range(5):
        frame(f)
    torch.cuda.synchronize()
    times = []
    for f in range(5, frames):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        frame(f)
        b.record(main)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    print(f"{name} K={K}: {np.median(times):.4f} ms/frame (median), rows {rows.tolist()}")
    for rd in ctxs:
        rd.close()
