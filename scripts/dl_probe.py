"""Experiment: where does the end-to-end frame time go?  Times, per frame at a
config (default C3): the graph-replayed render alone, the streamed G-buffer
download alone (bt_gbuffer_download_async + wait, no render), and both
interleaved as in bench.py's e2e pass."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200 import _capi as capi  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
s = Scene.build(name)
cfg = RenderConfig()
cam = s.device_camera
W, H = s.width, s.height
tx, ty = s.tiles
r = Renderer(0)
r.upload(s)
lib = r.lib
r.render_frame(cam, cfg, exact=False, graph=True)  # sizes the context

SPEC = ((W * H, torch.uint8), (W * H, torch.float32), (W * H * 3, torch.float32), (W * H, torch.int32),
        (tx * ty, torch.int32), (tx * ty, torch.int32), (tx * ty, torch.uint8))
off = (C.c_size_t * 7)()
total = C.c_size_t()
capi.check(lib.bt_gbuffer_layout(r.ctx, off, C.byref(total)), "layout")
slab_mode = len(sys.argv) > 2 and sys.argv[2] == "slab"


def host_set():
    if not slab_mode:  # seven separate pinned allocations: fourteen copies
        return [torch.empty(n, dtype=d).pin_memory() for n, d in SPEC]
    slab = torch.empty(total.value, dtype=torch.uint8).pin_memory()
    return [slab[off[i]:off[i] + n * torch.empty(0, dtype=d).element_size()] for i, (n, d) in enumerate(SPEC)]


outs = [host_set(), host_set()]


def dl(i):
    if slab_mode:
        capi.check(lib.bt_gbuffer_download_async_slab(r.ctx, C.c_void_p(outs[i % 2][0].data_ptr())), "dl")
    else:
        capi.check(lib.bt_gbuffer_download_async(r.ctx, *[C.c_void_p(t.data_ptr()) for t in outs[i % 2]]), "dl")


def timeit(fn, reps=40):
    for i in range(5):
        fn(i)
    capi.check(lib.bt_download_wait(r.ctx), "wait")
    capi.check(lib.bt_sync(r.ctx), "sync")
    t = time.perf_counter()
    for i in range(reps):
        fn(i)
    capi.check(lib.bt_download_wait(r.ctx), "wait")
    capi.check(lib.bt_sync(r.ctx), "sync")
    return (time.perf_counter() - t) / reps * 1e3


render = timeit(lambda i: r.render_frame(cam, cfg, exact=False, graph=True))
down = timeit(dl)


def both(i):
    r.render_frame(cam, cfg, exact=False, graph=True)
    dl(i)


e2e = timeit(both)
frames = [tuple(torch.from_numpy(a.view(np.int32) if a.dtype != np.float32 else a).pin_memory() for a in s.perturb(f))
          for f in range(4)]


def with_params(i):
    w, p, c = frames[i % 4]
    capi.check(lib.bt_params_update(r.ctx, C.c_void_p(w.data_ptr()), C.c_void_p(p.data_ptr()),
                                    C.c_void_p(c.data_ptr()), len(s.prims), 17), "params")
    both(i)


e2e_p = timeit(with_params)
mb = sum(t.numel() * t.element_size() for t in outs[0]) / 1e6
print(f"{name} ({'slab' if slab_mode else 'planes'}): render {render:.4f} ms | download alone {down:.4f} ms ({mb / down:.1f} GB/s for {mb:.1f} MB) | "
      f"render+download {e2e:.4f} ms ({W * H / e2e / 1e3:.0f} Mrays/s) | "
      f"host params+render+download {e2e_p:.4f} ms ({W * H / e2e_p / 1e3:.0f} Mrays/s)")
