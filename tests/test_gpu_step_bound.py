"""View-local step bound (bt_set_step_bound(ctx, 1)) against the reference.

Extension of the paper's ray processing (PAPER.md "Ray processing":
segment tracing "would provide a more robust solution"; conclusion:
"more advanced iterative ray processing, such as segment-tracing"): an
interval whose pruned view is 1-Lipschitz -- exact distances (sphere,
torus, box, sphere-cone) under sharp CSG -- is marched with L = 1 instead of
the global 1.45, so its steps are 1.45x longer; every other view keeps
the global bound.  The trajectory differs from the reference's, so this mode
has its own tolerance contract (the default mode 0 stays bit-exact):

  hit mask agreement >= 99.9 %; matched depth |dt| <= 2 minStep on >= 99.9 %
  and RMS <= 2 minStep over matched hits on the same surface; never more
  field evaluations than mode 0; normals (same hit mask, same surface):
  central-difference mode (a field gradient at the hit) dot >= 0.999 on
  >= 99.5 %; depth-differential mode dot >= 0.95 on >= 97 % -- a different
  march lands elsewhere inside the f <= hitEpsilon band (|dt| up to ~2e-3),
  and differencing neighbouring depths over a pixel footprint of ~1e-2 scene
  units turns that into normal noise (measured: C3 99.9 %, C1 99.0 %,
  random:64 97.6 % at 0.95).

Measured field evaluations saved by mode 1: C1 19.8 %, random:64 5.7 %,
gen:grid 5.0 %, C3 3.9 %, C2 / C5 < 0.5 % (their views blend almost
everywhere the rays march).
"""
import numpy as np
import pytest

from oracle_bridge import RefScene, ref_available
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def rd():
    r = Renderer(0)
    yield r
    r.close()


@pytest.mark.parametrize("mode", [0, 1])  # the normals mode
@pytest.mark.parametrize("name,w,h", [("C1", 0, 0), ("C2", 0, 0), ("C3", 0, 0), ("C5", 0, 0), ("random:64", 512, 512),
                                      ("gen:grid:2:mixed:smooth", 0, 0)])
def test_view_local_bound_against_reference(rd, name, w, h, mode):
    seed = 7 if name.startswith("gen") else 0
    cfg = RenderConfig()
    cfg.normalsMode = mode
    s = Scene.build(name, seed, w, h)
    gr, _, _, _ = RefScene(name, seed, w, h).frame(cfg, 0)
    rd.upload(s)
    evals = {}
    out = {}
    for sb in (0, 1):
        rd.set_step_bound(sb)
        rd.reset_stats()
        rd.render_frame(s.device_camera, cfg, exact=False, graph=False)
        out[sb] = rd.download_gbuffer()
        evals[sb] = rd.stats().fieldEvals
    rd.set_step_bound(0)
    g = out[1]
    m = (gr.hit == 1) & (g.hit == 1)
    dt = np.abs(gr.depth[m].astype(np.float64) - g.depth[m])
    near = dt <= 2 * cfg.minStep
    dots = (gr.normal[m] * g.normal[m]).sum(1)
    rep = {"hit": float((gr.hit == g.hit).mean()), "near": float(near.mean()) if len(dt) else 1.0,
           "rms": float(np.sqrt(np.mean(dt[near] ** 2))) if near.any() else 0.0,
           "dot": float((dots >= 0.999).mean()) if len(dots) else 1.0,
           "dot99": float((dots >= 0.99).mean()) if len(dots) else 1.0,
           "dot95": float((dots >= 0.95).mean()) if len(dots) else 1.0, "evals0": evals[0], "evals1": evals[1],
           "saved": 1.0 - evals[1] / max(1, evals[0])}
    print(name, rep)
    assert rep["hit"] >= 0.999, rep
    assert rep["near"] >= 0.999, rep
    assert rep["rms"] <= 2 * cfg.minStep, rep
    if mode == 1:
        assert rep["dot"] >= 0.995, rep
    else:
        assert rep["dot95"] >= 0.97, rep
    assert evals[1] <= evals[0], rep
