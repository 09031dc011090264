"""GPU tree compile (bt_tree_compile) against the
reference's compile (linear_tree.cpp:70-148).

Every scene's tree here was compiled on the host by the same source the
reference runs (tests/test_scenes.py pins the word arrays to the reference
bit for bit).  Its scene graph is recovered from the tree, shuffled into a
random node order, and compiled on the GPU: the words, the node records and
the primitive words must equal the host compile's bit for bit, and a frame
rendered from the GPU-compiled tree (its side tables built on the device)
must equal the reference's frame bit for bit.
"""
import numpy as np
import pytest

from oracle_bridge import RefScene, ref_available
from paper_2304_09673_b200.pipeline import GRAPH_DTYPE, RenderConfig, Renderer, Scene

pytestmark = pytest.mark.gpu

SCENES = [("C1", 0, 0, 0), ("C2", 0, 0, 0), ("C3", 0, 0, 0), ("C4", 0, 0, 0), ("C5", 0, 0, 0), ("csg", 0, 0, 0),
          ("random:200", 9, 256, 256), ("quad:60", 0, 0, 0), ("gen:grid:2:mixed:smooth", 7, 0, 0),
          ("comb_error", 0, 0, 0), ("sphere", 0, 0, 0)]


@pytest.fixture(scope="module")
def rd():
    r = Renderer(0)
    yield r
    r.close()


def plain_words(s: Scene) -> np.ndarray:
    """The scene's words as compile() emitted them: every blob's ancestor
    field is the parent's word (the scenes library then ran
    compute_fast_indices, which the node records' parentWord does not see)."""
    d = s.data.view(np.uint32).copy()
    for rec in s.nodes:
        b = d[4 * rec["word"]]
        d[4 * rec["word"]] = (b & ~np.uint32(0x7FFFFF)) | np.uint32(rec["parentWord"])
    return d


@pytest.mark.parametrize("name,seed,w,h", SCENES)
@pytest.mark.parametrize("order", [None, 1, 2])
def test_gpu_compile_equals_host_compile(rd, name, seed, w, h, order):
    s = Scene.build(name, seed, w, h)
    g, root = s.graph(order)
    rd.compile_tree(g, root)
    data, nodes, prims = rd.tree_arrays()
    assert data.view(np.uint32).tobytes() == plain_words(s).tobytes(), "tree words"
    assert nodes.tobytes() == s.nodes.tobytes(), "node records"
    assert prims.tobytes() == s.prims.tobytes(), "primitive words"
    # + compute_fast_indices on the device == the scene's own (host) fast indices
    rd.fast_indices()
    data, _, _ = rd.tree_arrays()
    assert data.view(np.uint32).tobytes() == s.data.view(np.uint32).tobytes(), "fast indices"


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,seed,w,h", [("C2", 0, 0, 0), ("C3", 0, 0, 0), ("C5", 0, 0, 0),
                                           ("random:200", 9, 256, 256)])
def test_frame_from_gpu_compiled_tree_equals_reference(rd, name, seed, w, h):
    cfg = RenderConfig()
    s = Scene.build(name, seed, w, h)
    g, root = s.graph(5)
    rd.scene = s
    rd.compile_tree(g, root)
    rd.fast_indices()  # the reference scene's tree carries fast indices
    rd.render_frame(s.device_camera, cfg, exact=True, graph=True)
    out = rd.download_gbuffer()
    gr, _, _, _ = RefScene(name, seed, w, h).frame(cfg, 0)
    for plane in ("hit", "depth", "normal", "evalCount", "tileMaxOverlap", "tileCacheBytes", "tileError"):
        assert np.ascontiguousarray(getattr(out, plane)).tobytes() == \
            np.ascontiguousarray(getattr(gr, plane)).tobytes(), plane


def test_gpu_compile_from_device_memory(rd):
    import torch
    s = Scene.build("C3")
    g, root = s.graph(11)
    dg = torch.from_numpy(g.view(np.uint8)).cuda()
    rd.compile_tree((dg.data_ptr(), len(g)), root, on_device=True)
    torch.cuda.synchronize()
    data, nodes, _ = rd.tree_arrays()
    assert data.view(np.uint32).tobytes() == plain_words(s).tobytes()
    assert nodes.tobytes() == s.nodes.tobytes()


def _bad(g, root, rd, what):
    with pytest.raises(Exception) as e:
        rd.compile_tree(g, root)
    assert what in str(e.value), str(e.value)


def test_gpu_compile_rejects_what_compile_rejects(rd):
    s = Scene.build("C1")
    g, root = s.graph(2)
    ops = np.nonzero(g["isPrimitive"] == 0)[0]
    prims = np.nonzero(g["isPrimitive"] == 1)[0]
    b = g.copy()
    b["left"][ops[0]] = -1
    _bad(b, root, rd, "two children")
    b = g.copy()
    b["right"][ops[0]] = b["left"][ops[1]]  # a node with two parents
    _bad(b, root, rd, "tree")
    b = g.copy()
    _bad(b, int(prims[0]), rd, "one tree")  # not the root
    b = g.copy()
    b["params"][prims[0]][7] = -1.0  # negative radius
    _bad(b, root, rd, "parameters")
    b = g.copy()
    b["params"][prims[1]][3] = 2.0  # not a unit quaternion
    _bad(b, root, rd, "parameters")
    b = g.copy()
    b["kind"][ops[0]] = 1  # not an operator kind
    _bad(b, root, rd, "kind")
    # a valid graph still compiles afterwards
    rd.compile_tree(g, root)
    data, _, _ = rd.tree_arrays()
    assert data.view(np.uint32).tobytes() == plain_words(s).tobytes()
