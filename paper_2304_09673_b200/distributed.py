"""Multi-GPU partition of the frame by screen-tile rows.

Tiles never interact in stages (b) and (c) (reference src/tracer.cpp:155-232),
so each rank builds the A-buffer of, and traces, only its contiguous range of
tile rows; the tree and the volumes are replicated (<= 1 MB).  There is no
collective on the tracing path: the only exchange is one gather of the
G-buffer rows to rank 0 after tracing, after which rank 0 computes the
depth-differential normals over the whole image (they need neighbour depths
across the row-range borders).

The gather works on torch tensors, so it runs with NCCL on device memory
(the context's own G-buffer planes, wrapped zero-copy) and with gloo on CPU
tensors in the multi-process tests.
"""
from __future__ import annotations

import numpy as np


def tile_row_ranges(tiles_y: int, world: int, row_cost: np.ndarray | None = None) -> np.ndarray:
    """Contiguous tile-row ranges, one per rank: returns world+1 row bounds.

    Without costs the rows are split evenly; with per-row costs (e.g. the
    A-buffer fragment count of each tile row from the previous frame) the
    split equalises the prefix sums.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    if row_cost is None or float(np.sum(row_cost)) <= 0.0:
        return np.linspace(0, tiles_y, world + 1).round().astype(np.int64)
    c = np.concatenate([[0.0], np.cumsum(np.asarray(row_cost, np.float64))])
    targets = np.linspace(0.0, c[-1], world + 1)
    bounds = np.searchsorted(c, targets[1:-1], side="left")
    out = np.concatenate([[0], bounds, [tiles_y]]).astype(np.int64)
    return np.maximum.accumulate(np.clip(out, 0, tiles_y))


def row_costs(eval_count: np.ndarray, width: int, height: int) -> np.ndarray:
    """March cost of every tile row: the field evaluations of its pixels
    (the G-buffer's evalCount plane of one full frame).  Feeding it to
    tile_row_ranges balances the ranks' marches -- the frame's dominant
    stage -- instead of their row counts."""
    ev = np.asarray(eval_count, np.float64).reshape(height, width).sum(axis=1)
    tiles_y = (height + 7) // 8
    out = np.zeros(tiles_y, np.float64)
    np.add.at(out, np.arange(height) // 8, ev)
    return out


def pixel_span(rows: np.ndarray, rank: int, width: int, height: int) -> tuple[int, int]:
    """[lo, hi) pixel-index range of rank's tile rows (row-major image)."""
    lo = int(min(rows[rank] * 8, height)) * width
    hi = int(min(rows[rank + 1] * 8, height)) * width
    return lo, hi


def gather_rows(planes: dict, rows: np.ndarray, rank: int, world: int, width: int, height: int,
                group=None) -> None:
    """Gather every rank's pixel rows of each plane into rank 0's planes.

    planes: name -> 1-D torch tensor over the full image (element per pixel,
    or `k` elements per pixel for vector planes of length k*width*height).
    Non-root ranks only need their own rows filled.
    """
    import torch
    import torch.distributed as dist

    spans = [pixel_span(rows, r, width, height) for r in range(world)]
    maxpx = max(hi - lo for lo, hi in spans)
    for name in sorted(planes):
        t = planes[name]
        per = t.numel() // (width * height)
        lo, hi = spans[rank]
        send = torch.zeros(maxpx * per, dtype=t.dtype, device=t.device)
        send[: (hi - lo) * per] = t[lo * per: hi * per]
        recv = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
        dist.gather(send, recv, dst=0, group=group)
        if rank == 0:
            for r, (a, b) in enumerate(spans):
                if r == 0:
                    continue
                t[a * per: b * per] = recv[r][: (b - a) * per]


class DeviceBytes:
    """Zero-copy __cuda_array_interface__ view of device memory."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def gbuffer_planes(view, device) -> dict:
    """Torch views of a context's device G-buffer (bt_gbuffer_view)."""
    import torch
    n = view.width * view.height
    return {
        "hit": torch.as_tensor(DeviceBytes(view.hit, n, "|u1"), device=device),
        "depth": torch.as_tensor(DeviceBytes(view.depth, n, "<f4"), device=device),
        "evalCount": torch.as_tensor(DeviceBytes(view.evalCount, n, "<i4"), device=device),
    }
