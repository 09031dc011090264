"""GPU tree compile (bt_tree_compile) time on the bench trees, the scene
graph resident in device memory (a structure edit made on the GPU), and the
device compute_fast_indices after it.  Wall clock around synchronous calls
(each returns after its readbacks), median of 20.

    python scripts/compile_bench.py [C3 C4 C5 ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_09673_b200.pipeline import Renderer, Scene  # noqa: E402

rd = Renderer(0)
for name in sys.argv[1:] or ["C3", "C4", "C5"]:
    s = Scene.build(name)
    g, root = s.graph(1)
    dg = torch.from_numpy(g.view(np.uint8)).cuda()
    torch.cuda.synchronize()
    tc, tf = [], []
    for _ in range(23):
        t0 = time.perf_counter()
        rd.compile_tree((dg.data_ptr(), len(g)), root, on_device=True)
        t1 = time.perf_counter()
        rd.fast_indices()
        rd.tree_arrays()  # (synchronises)
        t2 = time.perf_counter()
        tc.append(t1 - t0)
        tf.append(t2 - t1)
    print(f"{name}: {len(g)} nodes, GPU compile {np.median(tc[3:]) * 1e3:.3f} ms, "
          f"+ fast indices + download {np.median(tf[3:]) * 1e3:.3f} ms")
rd.close()
