"""One rank's share of an N-way tile-row split, eager frames (for an ncu
launch list of a single rank's kernels).  usage: shard_rank.py CONFIG N RANK [FRAMES]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200 import _capi as capi  # noqa: E402
from paper_2304_09673_b200.distributed import tile_row_ranges  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

name, n, rank = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
frames = int(sys.argv[4]) if len(sys.argv) > 4 else 3
s = Scene.build(name)
cfg, cam = RenderConfig(), s.device_camera
tx, ty = s.tiles
rows = tile_row_ranges(ty, n)
t0, t1 = int(rows[rank] * tx), int(rows[rank + 1] * tx)
rd = Renderer(0)
rd.upload(s)
for _ in range(frames):
    rd.render_frame(cam, cfg, exact=False, graph=False, tile0=t0, tile1=t1, normals=False)
capi.check(rd.lib.bt_sync(rd.ctx), "sync")
print(name, f"rank {rank}/{n}: tiles [{t0}, {t1})")
