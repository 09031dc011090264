"""Fused gather over peer memory (bt_gbuffer_export / bt_gbuffer_import):
the ranks trace contiguous ranges of tile rows; every non-root rank's march
writes its pixels and tile planes straight into rank 0's G-buffer (CUDA
IPC), and every rank then shades the normals of its OWN rows into rank 0's
normal plane (bt_normals_rows: the one-row depth halo across a row-range
border is read from rank 0's planes).  Run as a real multi-process job
(gloo for the handle exchange and the barriers) on ONE GPU -- the same IPC
mapping the multi-GPU path uses over NVLink.

Checked: the assembled frame equals a single-context render bit for bit
(exact mode), eagerly and through graph replays, over perturbed frames
(the bench's per-frame parameter updates), at 2 and 3 ranks."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PLANES = (("hit", "hit"), ("depth", "depth"), ("evalCount", "evalCount"), ("normal", "normal"),
          ("tmo", "tileMaxOverlap"), ("tcb", "tileCacheBytes"), ("terr", "tileError"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path, frames):
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
    for i, f in enumerate(frames):
        w, p, c = s.perturb(f)
        rd.update_params(w, p, c)
        rd.render_frame(cam, cfg, exact=True, graph=i > 0, tile0=t0, tile1=t1, normals=False)
        rd.sync()
        dist.barrier()  # every rank's rows are in rank 0's G-buffer
        rd.compute_normals_rows(cam, t0, t1, cfg.normalsMode, True)
        rd.sync()
        dist.barrier()  # every rank's normals are in rank 0's normal plane
        if rank == 0 and i == len(frames) - 1:
            g = rd.download_gbuffer()
            np.savez(out_path, hit=g.hit, depth=g.depth, evalCount=g.evalCount, normal=g.normal,
                     tmo=g.tileMaxOverlap, tcb=g.tileCacheBytes, terr=g.tileError)
        dist.barrier()  # rank 0 has read the frame: the next frame's peer writes may land
    if rank != 0:
        assert rd.lib.bt_gbuffer_import_release(rd.ctx) == 0
    dist.barrier()
    rd.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_gather_ranks_one_gpu(tmp_path, world):
    import torch.multiprocessing as mp

    from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene
    frames = [5, 6, 7]  # eager, capture, pure replay -- each a perturbed frame
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(_worker, args=(world, _free_port(), out, frames), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    s = Scene.build("C3")
    rd = Renderer(0)
    rd.upload(s)
    w, p, c = s.perturb(frames[-1])
    rd.update_params(w, p, c)
    rd.render_frame(s.device_camera, RenderConfig(), exact=True, graph=False)
    ref = rd.download_gbuffer()
    for k, plane in PLANES:
        assert got[k].tobytes() == getattr(ref, plane).tobytes(), k
