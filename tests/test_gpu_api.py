"""GPU behaviour of the boundary (run with -m gpu): the reference's own unit
tests against this library, graph replay, tile-range sharding, per-frame
parameter updates, the brute-force oracle, tile errors and determinism."""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle_bridge import Port, RefScene, compare_gbuffers, ref_available
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rd():
    r = Renderer(0)
    yield r
    r.close()


def test_reference_unit_tests_pass_against_b200_library():
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests_b200")
    if not os.path.exists(exe):
        pytest.skip("built only where /root/reference exists")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", p.stdout)
    assert m and m.group(1) == "72" and m.group(2) == "72", p.stdout + p.stderr[-3000:]


@pytest.mark.parametrize("exact", [True, False])
def test_graph_replay_equals_eager(rd, exact):
    cfg = RenderConfig()
    s = Scene.build("C3")
    rd.upload(s)
    rd.render_frame(s.device_camera, cfg, exact=exact, graph=False)
    a = rd.download_gbuffer()
    for _ in range(3):
        rd.render_frame(s.device_camera, cfg, exact=exact, graph=True)
    b = rd.download_gbuffer()
    for plane in ("hit", "depth", "evalCount", "normal", "tileMaxOverlap", "tileCacheBytes", "tileError"):
        assert getattr(a, plane).tobytes() == getattr(b, plane).tobytes(), plane


@pytest.mark.parametrize("name,parts", [("C3", 3), ("C4", 4)])
def test_tile_range_sharding_equals_full_frame(rd, name, parts):
    """Multi-GPU partition, on one device: tracing tile-row ranges separately
    reproduces the full frame (tiles never interact)."""
    cfg = RenderConfig()
    s = Scene.build(name)
    rd.upload(s)
    cam = s.device_camera
    rd.render_frame(cam, cfg, exact=False, graph=False)
    full = rd.download_gbuffer()
    tx, ty = s.tiles
    rows = np.linspace(0, ty, parts + 1).round().astype(int)
    rd.build_volumes_of_interest(cfg.hitEpsilon)
    for r in range(parts):
        t0, t1 = int(rows[r] * tx), int(rows[r + 1] * tx)
        rd.rasterize_volumes(cam, t0, t1)  # A-buffer of this shard only
        rd.render_tiles(cam, cfg, exact=False, tile0=t0, tile1=t1)
        part = rd.download_gbuffer()
        lo, hi = rows[r] * 8 * s.width, min(rows[r + 1] * 8, s.height) * s.width
        assert part.hit[lo:hi].tobytes() == full.hit[lo:hi].tobytes()
        assert part.depth[lo:hi].tobytes() == full.depth[lo:hi].tobytes()
        assert part.evalCount[lo:hi].tobytes() == full.evalCount[lo:hi].tobytes()


def test_per_frame_parameter_updates_match_reference(rd):
    cfg = RenderConfig()
    s = Scene.build("C3")
    rd.upload(s)
    cam = s.device_camera
    ref = RefScene("C3") if ref_available() else None
    for f in (1, 2):
        words, params, counts = s.perturb(f)
        rd.update_params(words, params, counts)
        assert rd.tree_words().tobytes() == s.data.tobytes()  # device words == host update_primitive_params
        rd.render_frame(cam, cfg, exact=True, graph=True)
        g = rd.download_gbuffer()
        if ref is not None:
            ref.perturb(f)
            gr, _, _, _ = ref.frame(cfg)
        else:
            gr, _, _, _ = Port.from_scene(s).frame(cfg, threads=os.cpu_count() or 4)
        assert g.hit.tobytes() == gr.hit.tobytes()
        assert g.depth.tobytes() == gr.depth.tobytes()
        assert g.normal.tobytes() == gr.normal.tobytes()


def test_oracle_render_and_pipeline_agree(rd):
    """test_tracer.cpp:226-247: pipeline vs brute-force oracle on a CSG scene."""
    cfg = RenderConfig()
    s = Scene.build("csg")
    rd.upload(s)
    cam = s.device_camera
    rd.oracle_render(cam, cfg, exact=True)
    go = rd.download_gbuffer()
    rd.render_frame(cam, cfg, exact=False, graph=False)
    gp = rd.download_gbuffer()
    if ref_available():
        rep = compare_gbuffers(gp, go, 2 * cfg.minStep)
        assert rep["hitAgreement"] >= 0.995 and rep["depthRms"] <= 2 * cfg.minStep
    m = (go.hit == 1) & (gp.hit == 1)
    assert (go.hit == gp.hit).mean() >= 0.995
    assert np.sqrt(np.mean((go.depth[m].astype(np.float64) - gp.depth[m]) ** 2)) <= 2 * cfg.minStep


def test_oracle_render_c1_matches_reference(rd):
    cfg = RenderConfig()
    s = Scene.build("C1", 0, 128, 128)
    rd.upload(s)
    rd.reset_stats()
    rd.oracle_render(s.device_camera, cfg, exact=True)
    g = rd.download_gbuffer()
    st = rd.stats()
    go, so = (RefScene("C1", 0, 128, 128).oracle(cfg) if ref_available()
              else Port.from_scene(s).oracle(cfg, threads=os.cpu_count() or 4))
    assert g.hit.tobytes() == go.hit.tobytes() and g.depth.tobytes() == go.depth.tobytes()
    assert g.evalCount.tobytes() == go.evalCount.tobytes()


def test_tile_errors_mark_tiles_and_render_continues(rd):
    """test_tracer.cpp:249-266: a 25-deep right comb overflows the stack."""
    cfg = RenderConfig()
    s = Scene.build("comb_error")
    rd.upload(s)
    rd.render_frame(s.device_camera, cfg, exact=True, graph=False)
    g = rd.download_gbuffer()
    assert g.tileError.any() and not g.tileError.all()
    assert rd.stats().tileErrors == int(g.tileError.sum())


def test_render_is_deterministic(rd):
    cfg = RenderConfig()
    s = Scene.build("C5")
    rd.upload(s)
    outs = []
    for _ in range(2):
        rd.render_frame(s.device_camera, cfg, exact=False, graph=False)
        g = rd.download_gbuffer()
        off, frags = rd.download_abuffer()
        outs.append((g.hit.tobytes(), g.depth.tobytes(), g.evalCount.tobytes(), off.tobytes(), frags.tobytes()))
    assert outs[0] == outs[1]


def test_c4_exact_vs_fast_agreement(rd):
    cfg = RenderConfig()
    s = Scene.build("C4")
    rd.upload(s)
    rd.render_frame(s.device_camera, cfg, exact=True, graph=False)
    ge = rd.download_gbuffer()
    rd.render_frame(s.device_camera, cfg, exact=False, graph=True)
    gf = rd.download_gbuffer()
    assert (ge.hit == gf.hit).mean() >= 0.999
    assert ge.hit.sum() > 0.2 * len(ge.hit)


def test_central_difference_normals_exact(rd):
    cfg = RenderConfig(normalsMode=1)
    s = Scene.build("csg", 0, 64, 64)
    rd.upload(s)
    rd.render_frame(s.device_camera, cfg, exact=True, graph=False)
    g = rd.download_gbuffer()
    gr, _, _, _ = (RefScene("csg", 0, 64, 64).frame(cfg) if ref_available()
                   else Port.from_scene(s).frame(cfg, threads=4))
    assert g.normal.tobytes() == gr.normal.tobytes()


def test_invalid_config_raises_before_device(rd):
    s = Scene.build("sphere")
    rd.upload(s)
    with pytest.raises(ValueError, match="relaxation"):
        rd.render_frame(s.device_camera, RenderConfig(relax=2.5))


def test_external_torch_stream(rd):
    import torch
    cfg = RenderConfig()
    s = Scene.build("C1")
    rd.upload(s)
    st = torch.cuda.Stream()
    rd.set_stream(st.cuda_stream)
    with torch.cuda.stream(st):
        rd.render_frame(s.device_camera, cfg, exact=True, graph=True)
    st.synchronize()
    g = rd.download_gbuffer()
    rd.set_stream(0)
    rd.render_frame(s.device_camera, cfg, exact=True, graph=False)
    assert rd.download_gbuffer().hit.tobytes() == g.hit.tobytes()


def test_streaming_download_matches_blocking_download(rd):
    """bt_gbuffer_download_async (device snapshot + copy stream, two slots):
    every frame of a perturbed sequence reaches the host intact, identical to
    a blocking download of the same frame."""
    import ctypes as C

    import torch
    cfg = RenderConfig()
    s = Scene.build("C1")
    rd.upload(s)
    cam = s.device_camera
    W, H = s.width, s.height
    tx, ty = s.tiles

    def planes():
        return [torch.zeros(n, dtype=d).pin_memory() for n, d in
                ((W * H, torch.uint8), (W * H, torch.float32), (W * H * 3, torch.float32), (W * H, torch.int32),
                 (tx * ty, torch.int32), (tx * ty, torch.int32), (tx * ty, torch.uint8))]
    streamed, reference = [], []
    for f in range(5):
        w, p, c = s.perturb(f)
        rd.update_params(w, p, c)
        rd.render_frame(cam, cfg, exact=False, graph=True)
        out = planes()
        assert rd.lib.bt_gbuffer_download_async(rd.ctx, *[C.c_void_p(t.data_ptr()) for t in out]) == 0
        streamed.append(out)
        g = rd.download_gbuffer()  # blocking; stream-ordered after the snapshot
        reference.append(g)
    assert rd.lib.bt_download_wait(rd.ctx) == 0
    for out, g in zip(streamed, reference):
        assert out[0].numpy().tobytes() == g.hit.tobytes()
        assert out[1].numpy().tobytes() == g.depth.tobytes()
        assert out[2].numpy().tobytes() == g.normal.tobytes()
        assert out[3].numpy().tobytes() == g.evalCount.tobytes()
        assert out[4].numpy().tobytes() == g.tileMaxOverlap.tobytes()
        assert out[6].numpy().tobytes() == g.tileError.tobytes()
    assert any(a.depth.tobytes() != b.depth.tobytes() for a, b in zip(reference, reference[1:])), "frames differ"


@pytest.mark.parametrize("w,h", [(512, 512), (203, 117)])
def test_streaming_download_into_one_slab(rd, w, h):
    """bt_gbuffer_download_async_slab: planes at bt_gbuffer_layout's offsets
    of one pinned slab go down as merged runs (two copies): identical to the blocking download,
    including odd image sizes whose planes are not 16-byte multiples (their
    padding is never written), and the bytes between planes stay untouched."""
    import ctypes as C

    import torch
    cfg = RenderConfig()
    s = Scene.build("C1", 0, w, h)
    rd.upload(s)
    cam = s.device_camera
    rd.render_frame(cam, cfg, exact=False, graph=False)
    off = (C.c_size_t * 7)()
    total = C.c_size_t()
    assert rd.lib.bt_gbuffer_layout(rd.ctx, off, C.byref(total)) == 0
    tx, ty = s.tiles
    sizes = [w * h, w * h * 4, w * h * 12, w * h * 4, tx * ty * 4, tx * ty * 4, tx * ty]
    assert all(off[i] + sizes[i] <= (off[i + 1] if i < 6 else total.value) for i in range(7))
    assert all(o % 16 == 0 for o in off)
    slab = torch.full((total.value + 64,), 0xA5, dtype=torch.uint8).pin_memory()
    for f in range(3):
        wv, p, c = s.perturb(f)
        rd.update_params(wv, p, c)
        rd.render_frame(cam, cfg, exact=False, graph=True)
        assert rd.lib.bt_gbuffer_download_async_slab(rd.ctx, C.c_void_p(slab.data_ptr())) == 0
        g = rd.download_gbuffer()
        assert rd.lib.bt_download_wait(rd.ctx) == 0
        b = slab.numpy()
        planes = [g.hit, g.depth, g.normal, g.evalCount, g.tileMaxOverlap, g.tileCacheBytes, g.tileError]
        for i, pl in enumerate(planes):
            raw = np.ascontiguousarray(pl).tobytes()
            assert len(raw) == sizes[i]
            assert b[off[i]:off[i] + sizes[i]].tobytes() == raw, f"plane {i}"
            end = off[i + 1] if i < 6 else total.value + 64
            assert (b[off[i] + sizes[i]:end] == 0xA5).all(), f"padding after plane {i} written"


def test_params_update_from_pinned_host_equals_pageable(rd):
    """bt_params_update reads PINNED host buffers with the update kernel
    itself (no copy engine); pageable buffers are staged.  Both give the
    same tree words, frame after frame, and the same rendered frame."""
    import ctypes as C

    import torch
    s = Scene.build("C3", 0, 320, 180)
    cfg = RenderConfig()
    trees, frames = [], []
    for pinned in (False, True):
        rd.upload(s)
        for f in range(3):
            w, p, c = s.perturb(f)
            if pinned:
                tw, tp, tc = (torch.from_numpy(a.view(np.int32) if a.dtype != np.float32 else a).pin_memory()
                              for a in (w, p, c))
                assert rd.lib.bt_params_update(rd.ctx, C.c_void_p(tw.data_ptr()), C.c_void_p(tp.data_ptr()),
                                               C.c_void_p(tc.data_ptr()), len(w), 17) == 0
                assert rd.lib.bt_sync(rd.ctx) == 0  # the pinned buffers are read in stream order
            else:
                rd.update_params(w, p, c)
        trees.append(rd.tree_words())
        rd.render_frame(s.device_camera, cfg, exact=True, graph=False)
        frames.append(rd.download_gbuffer())
    assert trees[0].tobytes() == trees[1].tobytes()
    assert frames[0].depth.tobytes() == frames[1].depth.tobytes()


def test_frames_in_flight_equal_back_to_back_frames(rd):
    """Two contexts on their own streams rendering alternate frames of a
    perturbed sequence concurrently (bench.py's frames_in_flight) give the
    frames a single context renders back to back, bit for bit."""
    import torch
    s = Scene.build("C3", 0, 480, 270)
    cfg = RenderConfig()
    cam = s.device_camera
    seq = [s.perturb(f) for f in range(4)]
    ref = []
    rd.upload(s)
    for w, p, c in seq:
        rd.update_params(w, p, c)
        rd.render_frame(cam, cfg, exact=False, graph=True)
        ref.append(rd.download_gbuffer())
    streams = [torch.cuda.Stream() for _ in range(2)]
    ctxs = []
    for st in streams:
        r = Renderer(0)
        r.set_stream(st.cuda_stream)
        r.upload(s)
        ctxs.append(r)
    got = []
    try:
        for rnd in range(2):  # frames 0,1 concurrently, then 2,3
            for k in range(2):
                w, p, c = seq[2 * rnd + k]
                ctxs[k].update_params(w, p, c)
                ctxs[k].render_frame(cam, cfg, exact=False, graph=True)
            torch.cuda.synchronize()
            got += [ctxs[0].download_gbuffer(), ctxs[1].download_gbuffer()]
    finally:
        for r in ctxs:
            r.close()
    for a, b in zip(got, ref):
        assert a.depth.tobytes() == b.depth.tobytes() and a.normal.tobytes() == b.normal.tobytes()
        assert a.hit.tobytes() == b.hit.tobytes() and a.evalCount.tobytes() == b.evalCount.tobytes()


def test_march_schedule_never_changes_results(rd):
    """Raster order, the device's longest-first order with half-tile units
    (mode 1) and a random host permutation give bit-identical frames and
    RenderStats (tiles are independent; a tile's two halves walk prefixes of
    the same interval list).  Only the lockstep-step diagnostic may differ."""
    import ctypes as C
    cfg = RenderConfig()
    s = Scene.build("C3")
    rd.upload(s)
    cam = s.device_camera
    outs = []
    for mode in ("raster", "lpt", "random"):
        if mode == "raster":
            assert rd.lib.bt_set_scheduling(rd.ctx, 0) == 0
        elif mode == "lpt":
            assert rd.lib.bt_set_scheduling(rd.ctx, 1) == 0
        else:
            tx, ty = s.tiles
            perm = np.random.default_rng(7).permutation(tx * ty).astype(np.uint32)
            assert rd.lib.bt_set_tile_order(rd.ctx, perm.ctypes.data_as(C.c_void_p), len(perm)) == 0
        rd.reset_stats()
        rd.render_frame(cam, cfg, exact=True, graph=False)
        st = rd.stats()
        outs.append((rd.download_gbuffer(), (st.fieldEvals, st.retainedNodeVisits, st.primitiveEvals,
                                             st.maxOverlap, st.maxCacheBytes, st.tileErrors)))
    assert rd.lib.bt_set_scheduling(rd.ctx, 1) == 0
    base, bst = outs[0]
    for g, st in outs[1:]:
        assert st == bst
        for plane in ("hit", "depth", "evalCount", "normal", "tileMaxOverlap", "tileCacheBytes", "tileError"):
            assert getattr(g, plane).tobytes() == getattr(base, plane).tobytes(), plane


@pytest.mark.parametrize("name", ["C3", "C5", "comb_error", "random:24", "csg", "gen:cells:40:mixed:smooth"])
def test_device_fast_indices_equal_host(rd, name):
    """GPU tree preprocessing: a tree uploaded with plain
    parent ancestors, then bt_tree_fast_indices on the device, is bit-identical
    to the host compute_fast_indices result -- and renders identically."""
    seed = 7 if name.startswith("gen") else 0
    s = Scene.build(name, seed)
    fast = s.data.copy()
    data = s.data.copy()
    blobs = data.view(np.uint32)
    for n in s.nodes:  # blob ancestor := parent word (the root keeps the sentinel)
        w = int(n["word"]) * 4
        anc = int(n["parentWord"]) & 0x7FFFFF
        blobs[w] = (int(blobs[w]) & ~0x7FFFFF) | anc
    assert data.tobytes() != fast.tobytes() or name == "csg"
    s.data = data  # upload the parent-pointer tree
    rd.upload(s)
    s.data = fast
    assert rd.lib.bt_tree_fast_indices(rd.ctx) == 0
    got = rd.tree_words()
    assert got.view(np.uint32).tobytes() == fast.view(np.uint32).tobytes()
    cfg = RenderConfig()
    rd.render_frame(s.device_camera, cfg, exact=True, graph=False)
    a = rd.download_gbuffer()
    rd.upload(s)
    rd.render_frame(s.device_camera, cfg, exact=True, graph=False)
    b = rd.download_gbuffer()
    for plane in ("hit", "depth", "evalCount", "tileMaxOverlap", "tileCacheBytes", "tileError"):
        assert getattr(a, plane).tobytes() == getattr(b, plane).tobytes(), plane


def test_graph_replay_capacity_overflow_is_flagged_then_eager_frame_grows():
    """A graph is captured on a frame whose buffers fit (tiny primitives), then
    the parameters grow every primitive back (C4: 10,000 primitives at 4K) and
    the graph is replayed: the fragment store and the superblock candidate
    lists overflow.  The replay must stay in bounds and be flagged
    (bt_stats_download -> BT_ENOMEM), and the next eager frame must grow the
    buffers and render the frame bit-identically to a fresh context."""
    from paper_2304_09673_b200._capi import BtError
    cfg = RenderConfig()
    s = Scene.build("C4")
    w, p, c = s.perturb(1)
    small = p.copy()
    for i in range(len(c)):
        small[i, 7:c[i]] *= 0.02  # shape parameters (radii, extents) -- the transforms stay
    cam = s.device_camera
    rd = Renderer(0)
    fresh = Renderer(0)
    try:
        rd.upload(s)
        rd.update_params(w, small, c)
        rd.render_frame(cam, cfg, exact=False, graph=True)  # eager sizing on the small frame, then capture
        rd.stats()
        rd.update_params(w, p, c)
        rd.reset_stats()
        rd.render_frame(cam, cfg, exact=False, graph=True)  # replay of the small frame's graph
        with pytest.raises(BtError):
            rd.stats()
        rd.reset_stats()
        rd.render_frame(cam, cfg, exact=True, graph=False)  # checked: grows and renders
        g = rd.download_gbuffer()
        st = rd.stats()
        assert st.tileErrors == 0 and g.hit.any()
        fresh.upload(s)  # the scene's tree carries frame 1's parameters
        fresh.render_frame(cam, cfg, exact=True, graph=False)
        gf = fresh.download_gbuffer()
        for plane in ("hit", "depth", "evalCount", "normal", "tileMaxOverlap", "tileCacheBytes", "tileError"):
            assert getattr(g, plane).tobytes() == getattr(gf, plane).tobytes(), plane
        # and the graph path recovers: the next captured frame equals the eager one
        rd.render_frame(cam, cfg, exact=True, graph=True)
        assert rd.download_gbuffer().depth.tobytes() == gf.depth.tobytes()
        rd.stats()
    finally:
        rd.close()
        fresh.close()
