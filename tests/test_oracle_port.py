"""The C restatement (oracle/port/bt_port.c) against the unmodified
reference library on identical scenes: every stage bit-exact."""
import numpy as np
import pytest

from conftest import need_ref
from edge_cases import EDGE
from oracle_bridge import Port, RefScene
from paper_2304_09673_b200.pipeline import RenderConfig, Scene


def same(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.nbytes == b.nbytes and a.view(np.uint8).tobytes() == b.view(np.uint8).tobytes()


@pytest.mark.parametrize("name,w,h", [("sphere", 0, 0), ("csg", 0, 0), ("comb_error", 0, 0), ("random:24", 0, 0),
                                      ("C1", 256, 256), ("gen:grid:2:mixed:smooth", 160, 160),
                                      ("C5", 240, 136)])
def test_port_equals_reference(name, w, h):
    need_ref()
    cfg = RenderConfig()
    seed = 7 if name.startswith("gen") else 0
    s = Scene.build(name, seed, w, h)
    r = RefScene(name, seed, w, h)
    p = Port.from_scene(s)
    assert same(r.roi(), p.roi())
    vr, vp = r.vois(cfg.hitEpsilon), p.vois(cfg.hitEpsilon)
    assert same(vr, vp)
    offr, frr, _ = r.rasterize(vr)
    offp, frp = p.rasterize(vp)
    assert same(offr, offp) and same(frr, frp)
    gr, sr, _ = r.render_tiles(cfg, offr, frr, threads=4, normals=True)
    gp, sp = p.render_tiles(cfg, offp, frp, threads=4)
    p.normals(gp)
    for plane in ("hit", "depth", "evalCount", "normal", "tileMaxOverlap", "tileCacheBytes", "tileError"):
        assert same(getattr(gr, plane), getattr(gp, plane)), plane
    assert list(sp) == [sr.fieldEvals, sr.retainedNodeVisits, sr.primitiveEvals, sr.treeNodeCount, sr.maxOverlap,
                        sr.maxCacheBytes]


def test_port_oracle_render_equals_reference():
    need_ref()
    cfg = RenderConfig()
    s = Scene.build("csg", 0, 64, 64)
    r = RefScene("csg", 0, 64, 64)
    p = Port.from_scene(s)
    gr, sr = r.oracle(cfg, threads=4)
    gp, sp = p.oracle(cfg, threads=4)
    assert same(gr.hit, gp.hit) and same(gr.depth, gp.depth) and same(gr.evalCount, gp.evalCount)
    assert list(sp[:3]) == [sr.fieldEvals, sr.retainedNodeVisits, sr.primitiveEvals]


def test_central_difference_normals_equal_reference():
    need_ref()
    cfg = RenderConfig(normalsMode=1)
    s = Scene.build("csg", 0, 64, 64)
    r = RefScene("csg", 0, 64, 64)
    p = Port.from_scene(s)
    gr, _, _, _ = r.frame(cfg, threads=2)
    gp, _, _, _ = p.frame(cfg, threads=2)
    assert same(gr.normal, gp.normal)


@pytest.mark.parametrize("name,cam14,what", EDGE, ids=[e[2] for e in EDGE])
def test_port_equals_reference_edge_cameras(name, cam14, what):
    """The C restatement on degenerate cameras and images (no fragments,
    camera inside volumes, sub-tile images, overlap saturation)."""
    need_ref()
    cfg = RenderConfig()
    s = Scene.build(name)
    s.set_camera(cam14)
    r = RefScene(name)
    r.set_camera(cam14)
    p = Port.from_scene(s)
    vr, vp = r.vois(cfg.hitEpsilon), p.vois(cfg.hitEpsilon)
    assert same(vr, vp)
    offr, frr, _ = r.rasterize(vr)
    offp, frp = p.rasterize(vp)
    assert same(offr, offp) and same(frr, frp)
    gr, sr, _ = r.render_tiles(cfg, offr, frr, threads=4, normals=True)
    gp, sp = p.render_tiles(cfg, offp, frp, threads=4)
    p.normals(gp)
    for plane in ("hit", "depth", "evalCount", "normal", "tileMaxOverlap", "tileCacheBytes", "tileError"):
        assert same(getattr(gr, plane), getattr(gp, plane)), plane
    assert list(sp) == [sr.fieldEvals, sr.retainedNodeVisits, sr.primitiveEvals, sr.treeNodeCount, sr.maxOverlap,
                        sr.maxCacheBytes]


def test_invalid_scene_camera_is_rejected():
    s = Scene.build("sphere")
    with pytest.raises(ValueError):
        s.set_camera(np.array([0, 0, -6, 0, 0, 0, 0, 1, 0, 45, 0.1, 40, 0, 16], np.float32))  # width 0
