"""Host-side logic: config validation (same rules/messages as the
reference's validate_config), the multi-GPU tile-row partition and the
rank-0 gather, run as a real 2-process gloo job on CPU."""
import os
import socket

import numpy as np
import pytest

from paper_2304_09673_b200.distributed import gather_rows, pixel_span, tile_row_ranges
from paper_2304_09673_b200.pipeline import RenderConfig


@pytest.mark.parametrize("kw,msg", [({"relax": 2.0}, "relaxation"), ({"relax": 0.9}, "relaxation"),
                                    ({"lipschitz": 0.5}, "lipschitz"), ({"minStep": 0.0}, "min step"),
                                    ({"hitEpsilon": -1.0}, "hit epsilon"), ({"maxOverlap": 0}, "max overlap"),
                                    ({"maxOverlap": 97}, "max overlap")])
def test_config_validation_matches_reference(kw, msg):
    # reference src/tracer.cpp:10-19
    with pytest.raises(ValueError, match=msg):
        RenderConfig(**kw).to_c()


def test_default_config_constants():
    c = RenderConfig()
    assert np.float32(c.hitEpsilon) == np.float32(0.5) * np.float32(0.005) * np.float32(1.45)
    assert (c.lipschitz, c.relax, c.minStep, c.maxOverlap, c.maxNewPerFetch) == (1.45, 1.7, 0.005, 96, 6)


@pytest.mark.parametrize("tiles_y,world", [(135, 1), (135, 2), (135, 8), (270, 4), (7, 8)])
def test_tile_rows_cover_exactly(tiles_y, world):
    rows = tile_row_ranges(tiles_y, world)
    assert rows[0] == 0 and rows[-1] == tiles_y and len(rows) == world + 1
    assert (np.diff(rows) >= 0).all()
    assert np.diff(rows).max() - np.diff(rows).min() <= 1


def test_tile_rows_balance_costs():
    cost = np.zeros(100)
    cost[:10] = 100.0  # all the work at the top
    rows = tile_row_ranges(100, 4, cost)
    assert rows[0] == 0 and rows[-1] == 100 and (np.diff(rows) >= 0).all()
    shares = [cost[rows[i]:rows[i + 1]].sum() for i in range(4)]
    assert max(shares) <= 300.0


def test_pixel_spans_partition_the_image():
    rows = tile_row_ranges(135, 3)
    spans = [pixel_span(rows, r, 1920, 1080) for r in range(3)]
    assert spans[0][0] == 0 and spans[-1][1] == 1920 * 1080
    assert all(spans[i][1] == spans[i + 1][0] for i in range(2))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gather_worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, H = 40, 28  # 5 x 4 tiles (last tile row partial)
    tiles_y = (H + 7) // 8
    rows = tile_row_ranges(tiles_y, world)
    full_hit = (np.arange(W * H) % 3 == 0).astype(np.uint8)
    full_depth = np.arange(W * H, dtype=np.float32) * 0.25
    full_norm = np.arange(3 * W * H, dtype=np.float32)
    lo, hi = pixel_span(rows, rank, W, H)
    # each rank only renders its own rows (elsewhere: garbage)
    hit = np.full(W * H, 7, np.uint8)
    depth = np.full(W * H, -1.0, np.float32)
    norm = np.full(3 * W * H, -5.0, np.float32)
    hit[lo:hi], depth[lo:hi], norm[3 * lo:3 * hi] = full_hit[lo:hi], full_depth[lo:hi], full_norm[3 * lo:3 * hi]
    planes = {"hit": torch.from_numpy(hit), "depth": torch.from_numpy(depth), "normal": torch.from_numpy(norm)}
    gather_rows(planes, rows, rank, world, W, H)
    if rank == 0:
        ok = (planes["hit"].numpy() == full_hit).all() and (planes["depth"].numpy() == full_depth).all() and \
            (planes["normal"].numpy() == full_norm).all()
        open(out_path, "w").write("ok" if ok else "mismatch")
    dist.destroy_process_group()


def test_gather_rows_gloo_world2(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "result.txt")
    mp.spawn(_gather_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert open(out).read() == "ok"


def test_gather_rows_gloo_world3(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "result.txt")
    mp.spawn(_gather_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    assert open(out).read() == "ok"


def test_row_costs_balance_the_split():
    """row_costs sums each tile row's evaluations; the cost-balanced split
    puts more rows on the ranks whose rows are cheap."""
    from paper_2304_09673_b200.distributed import row_costs
    w, h = 64, 80  # 10 tile rows
    ev = np.zeros((h, w), np.uint32)
    ev[32:48, :] = 100  # tile rows 4 and 5 carry all the work
    c = row_costs(ev.reshape(-1), w, h)
    assert c.shape == (10,) and c[4] == c[5] == 100 * 8 * w and c.sum() == ev.sum()
    rows = tile_row_ranges(10, 2, c)
    assert rows[0] == 0 and rows[-1] == 10 and rows[1] == 5  # one heavy row per rank
