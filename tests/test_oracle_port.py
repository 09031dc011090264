"""The C restatement (oracle/port/bt_port.c) against the unmodified
reference library on identical scenes: every stage bit-exact."""
import numpy as np
import pytest

from conftest import need_ref
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
