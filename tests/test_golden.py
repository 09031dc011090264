"""The oracle is pinned: the reference's own known-answer values and the
golden scene fixtures (tests/golden/, generated from the unmodified
reference by tests/golden/make_golden.py) are reproduced bit for bit by the
C restatement (oracle/port) and, when built, by the reference itself."""
import ctypes as C
import glob
import os

import numpy as np
import pytest

from oracle_bridge import Port, RefScene, port_lib, ref_available
from paper_2304_09673_b200.pipeline import FRAG_DTYPE, VOI_DTYPE, RenderConfig, Scene, ptr

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SCENES = sorted(glob.glob(os.path.join(GOLDEN, "scene_*.npz")))


def test_field_known_answers():
    z = np.load(os.path.join(GOLDEN, "field_known_answers.npz"))
    lib = port_lib()
    for i in range(len(z["prim_kind"])):
        p = np.ascontiguousarray(z["prim_params"][i])
        v = lib.port_eval_primitive(int(z["prim_kind"][i]), ptr(p), *[C.c_float(x) for x in z["prim_point"][i]])
        # the restatement equals the reference bit for bit ...
        assert np.float32(v).view(np.uint32) == z["prim_ref"][i].view(np.uint32)
        # ... and both satisfy the reference tests' literal (test_field.cpp:47-72)
        exp, tol = z["prim_expected"][i], z["prim_tol"][i]
        assert abs(v - exp) <= tol * max(1.0, abs(exp)) + 1e-7
    for i in range(len(z["op_code"])):
        kd = np.ascontiguousarray(z["op_kd"][i])
        f0, f1 = z["op_f"][i]
        v = lib.port_eval_operator(int(z["op_code"][i]), ptr(kd), C.c_float(f0), C.c_float(f1))
        assert np.float32(v).view(np.uint32) == z["op_ref"][i].view(np.uint32)
        exp, tol = z["op_expected"][i], z["op_tol"][i]
        assert (v == exp) if np.isinf(exp) else abs(v - exp) <= tol + 1e-7


def load(path):
    z = np.load(path)
    name = str(z["name"])
    return z, name, int(z["width"]), int(z["height"])


@pytest.mark.parametrize("path", SCENES, ids=[os.path.basename(p) for p in SCENES])
def test_port_reproduces_golden_scene(path):
    z, name, w, h = load(path)
    cfg = RenderConfig()
    s = Scene.build(name, 0, w, h)
    port = Port.from_scene(s)
    assert port.roi().tobytes() == z["roi"].tobytes()
    vois = port.vois(cfg.hitEpsilon)
    assert vois.view(np.uint8).tobytes() == z["vois"].tobytes()
    off, frags = port.rasterize(vois)
    assert off.tobytes() == z["offsets"].tobytes()
    assert frags.view(np.uint8).tobytes() == z["frags"].tobytes()
    g, st = port.render_tiles(cfg, off, frags, threads=4)
    port.normals(g)
    for plane in ("hit", "depth", "evalCount", "normal", "tileMaxOverlap", "tileCacheBytes", "tileError"):
        assert getattr(g, plane).tobytes() == z[plane].tobytes(), plane
    assert list(st) == list(z["stats"])
    if "oracle_hit" in z:
        go, so = port.oracle(cfg, threads=4)
        assert go.hit.tobytes() == z["oracle_hit"].tobytes()
        assert go.depth.tobytes() == z["oracle_depth"].tobytes()
        assert go.evalCount.tobytes() == z["oracle_evalCount"].tobytes()
        assert list(so[:3]) == list(z["oracle_stats"])


@pytest.mark.parametrize("path", SCENES[:3], ids=[os.path.basename(p) for p in SCENES[:3]])
def test_reference_regenerates_golden_scene(path):
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    z, name, w, h = load(path)
    cfg = RenderConfig()
    r = RefScene(name, 0, w, h)
    g, st, _, _ = r.frame(cfg, threads=2)
    assert g.hit.tobytes() == z["hit"].tobytes() and g.depth.tobytes() == z["depth"].tobytes()
    assert g.normal.tobytes() == z["normal"].tobytes()
