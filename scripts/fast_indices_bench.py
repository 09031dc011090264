"""Device compute_fast_indices (bt_tree_fast_indices) time on the bench trees."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200.pipeline import Renderer, Scene  # noqa: E402

for name in sys.argv[1:] or ["C3", "C5", "C4"]:
    s = Scene.build(name)
    rd = Renderer(0)
    rd.upload(s)
    for _ in range(3):
        rd.lib.bt_tree_fast_indices(rd.ctx)
    rd.sync()
    t = time.perf_counter()
    for _ in range(20):
        rd.lib.bt_tree_fast_indices(rd.ctx)
    rd.sync()
    ms = (time.perf_counter() - t) / 20 * 1e3
    print(f"{name}: {len(s.nodes)} nodes, device compute_fast_indices {ms:.3f} ms (wall, incl. launches)")
    rd.close()
