"""Fused gather over peer memory (bt_gbuffer_export / bt_gbuffer_import):
two ranks trace the two halves of the tile rows; rank 1's march writes its
pixels and tile planes straight into rank 0's G-buffer (CUDA IPC).  Run as a
real 2-process job (gloo for the handle exchange and the barrier) on ONE GPU
-- the same IPC mapping the multi-GPU path uses over NVLink."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_2304_09673_b200 import _capi as capi
    from paper_2304_09673_b200.distributed import tile_row_ranges
    from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = Scene.build("C3")
    cfg, cam = RenderConfig(), s.device_camera
    tx, ty = s.tiles
    rows = tile_row_ranges(ty, world)
    t0, t1 = int(rows[rank] * tx), int(rows[rank + 1] * tx)
    rd = Renderer(0)
    rd.upload(s)
    rd.render_frame(cam, cfg, exact=True, graph=False, tile0=t0, tile1=t1, normals=False)  # allocates the planes
    h = capi.bt_ipc_handles()
    if rank == 0:
        assert rd.lib.bt_gbuffer_export(rd.ctx, C.byref(h)) == 0
    obj = [bytes(h)]
    dist.broadcast_object_list(obj, src=0)
    if rank != 0:
        C.memmove(C.addressof(h), obj[0], C.sizeof(h))
        assert rd.lib.bt_gbuffer_import(rd.ctx, C.byref(h)) == 0
    dist.barrier()
    for graph in (False, True):  # eager, then captured + replayed
        for _ in range(2 if graph else 1):
            rd.render_frame(cam, cfg, exact=True, graph=graph, tile0=t0, tile1=t1, normals=False)
        rd.sync()
        dist.barrier()  # every rank's tiles are in rank 0's G-buffer
    if rank == 0:
        rd.compute_normals(cam, cfg.normalsMode, True)
        g = rd.download_gbuffer()
        np.savez(out_path, hit=g.hit, depth=g.depth, evalCount=g.evalCount, normal=g.normal,
                 tmo=g.tileMaxOverlap, tcb=g.tileCacheBytes, terr=g.tileError)
    else:
        assert rd.lib.bt_gbuffer_import_release(rd.ctx) == 0
    dist.barrier()
    rd.close()
    dist.destroy_process_group()


def test_fused_gather_two_ranks_one_gpu(tmp_path):
    import torch.multiprocessing as mp

    from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    s = Scene.build("C3")
    rd = Renderer(0)
    rd.upload(s)
    rd.render_frame(s.device_camera, RenderConfig(), exact=True, graph=False)
    ref = rd.download_gbuffer()
    for k, plane in (("hit", "hit"), ("depth", "depth"), ("evalCount", "evalCount"), ("normal", "normal"),
                     ("tmo", "tileMaxOverlap"), ("tcb", "tileCacheBytes"), ("terr", "tileError")):
        assert got[k].tobytes() == getattr(ref, plane).tobytes(), k
