"""The workload recipes produce bit-identical compiled trees through this
repo's drop-in C++ API and through the unmodified reference API (same
source, same RNG draws), so every parity test compares identical inputs."""
import numpy as np
import pytest

from conftest import need_ref
from paper_2304_09673_b200.pipeline import Scene

SCENES = ["C1", "C2", "C3", "C4", "C5", "sphere", "csg", "slab", "comb_error", "random:24",
          "gen:cells:167:hex:smooth", "gen:grid:2:mixed:smooth", "gen:cells:334:tri:sharp"]


@pytest.mark.parametrize("name", SCENES)
def test_scene_identical_to_reference_build(name):
    need_ref()
    from oracle_bridge import RefScene
    seed = 7 if name.startswith("gen") else 0
    s = Scene.build(name, seed)
    r = RefScene(name, seed)
    data, nodes, prims = r.tree()
    assert s.data.view(np.uint32).tobytes() == data.view(np.uint32).tobytes()
    assert (s.nodes == nodes).all() and (s.prims == prims).all()
    assert (s.camera14 == r.camera14()).all()


def test_config_sizes():
    # primitive counts and resolutions
    want = {"C1": (10, 512, 512), "C2": (142, 1920, 1080), "C3": (1000, 1920, 1080), "C4": (10000, 3840, 2160),
            "C5": (4000, 1920, 1080)}
    for name, (n, w, h) in want.items():
        s = Scene.build(name)
        assert (len(s.prims), s.width, s.height) == (n, w, h)


def test_c5_is_deep():
    # depth >= 64: walk parent chains of the node records
    s = Scene.build("C5")
    word_to_ord = {int(w): i for i, w in enumerate(s.nodes["word"])}
    depth = 0
    for i in range(len(s.nodes)):
        d, cur = 0, i
        while s.nodes["parentWord"][cur] != 0x7FFFFF:
            cur = word_to_ord[int(s.nodes["parentWord"][cur])]
            d += 1
        depth = max(depth, d)
    assert depth >= 64


def test_perturbation_identical_to_reference():
    need_ref()
    from oracle_bridge import RefScene
    s = Scene.build("C3")
    r = RefScene("C3")
    for f in (0, 1, 7):
        words, params, counts = s.perturb(f)
        r.perturb(f)
        data, _, _ = r.tree()
        assert s.data.view(np.uint32).tobytes() == data.view(np.uint32).tobytes()
        assert len(words) == 1000 and (counts >= 8).all()
