"""Per-node cost of a CUDA graph of N dependent tiny kernels (torch add_ on
one element): bounds the launch-gap share of the frame graph."""
import time

import torch

x = torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
for n in (1, 10, 28, 56):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                x.add_(1)
    torch.cuda.synchronize()
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(200):
        g.replay()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 200 * 1e6
    print(f"graph of {n} dependent tiny kernels: {dt:.1f} us per replay, {dt / n:.2f} us per node")
