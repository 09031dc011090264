"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
(oracle/_ref/libbt_ref.so, built from /root/reference/proj/src).

    python tests/golden/make_golden.py

* field_known_answers.npz -- the known-answer field values of the
  reference's own tests (proj/tests/test_field.cpp:47-72,92-137), evaluated
  by the reference library, next to the literals those tests assert.
* scene_<name>.npz        -- per scene: VOIs, CSR A-buffer, full G-buffer and
  RenderStats of the reference pipeline (test_tracer.cpp:25-31 composition),
  plus oracle_render for the csg scene (test_tracer.cpp:226-247).
The fixtures travel to the GPU box (which has no /root/reference) and pin
both the C restatement and the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_bridge import RefScene, ref_lib  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, ptr  # noqa: E402

# scene name, width, height
GOLDEN_SCENES = [("sphere", 128, 128), ("csg", 128, 128), ("slab", 128, 128), ("comb_error", 64, 64),
                 ("random:24", 96, 96), ("C1", 160, 160), ("C2", 240, 136), ("C5", 192, 108)]


def prim_params(kind, t=(0.0, 0.0, 0.0), q=(1.0, 0.0, 0.0, 0.0), shape=()):
    p = np.zeros(17, np.float32)
    p[0:3] = t
    p[3:7] = q
    p[7:7 + len(shape)] = shape
    return p


def field_known_answers():
    """(kind, params, point, expected literal, tolerance) from test_field.cpp."""
    s, c = np.sin(np.float32(3.14159265 / 4)), np.cos(np.float32(3.14159265 / 4))
    rows = [
        (0, prim_params(0, shape=(1.0,)), (2, 0, 0), 1.0, 1e-6),                        # :48
        (0, prim_params(0, shape=(1.0,)), (0, 0, 0), -1.0, 1e-6),                       # :49
        (3, prim_params(3, shape=(1, 1, 1)), (2, 2, 0), float(np.sqrt(2.0)), 1e-4),     # :51-54
        (2, prim_params(2, shape=(2.0, 0.5)), (2, 0, 0), -0.5, 1e-6),                   # :57
        (2, prim_params(2, shape=(2.0, 0.5)), (4, 0, 0), 1.5, 1e-6),                    # :58
        (4, prim_params(4, shape=(0.5, 0.2, 1.0)), (0, -1, 0), 0.5, 1e-6),              # :61
        (4, prim_params(4, shape=(0.5, 0.2, 1.0)), (0, 2, 0), 0.8, 1e-6),               # :62
        (3, prim_params(3, t=(3, 0, 0), q=(c, 0, 0, s), shape=(2, 0.5, 0.5)), (3, 2, 0), 0.0, 1e-5),    # :66-70
        (3, prim_params(3, t=(3, 0, 0), q=(c, 0, 0, s), shape=(2, 0.5, 0.5)), (3.5, 0, 0), 0.0, 1e-5),  # :71
    ]
    ops = [  # code, k, d, f0, f1, expected, tol (test_field.cpp:73-137)
        (3, 0, 0, 1.0, 2.0, 1.0, 0.0), (4, 0, 0, -0.5, 0.2, 0.2, 0.0), (5, 0, 0, 0.5, -0.2, 0.5, 0.0),
        (6, 1.0, 0, 0.0, 0.0, -1.0 / 6.0, 1e-6), (7, 1.0, 0, 0.0, 0.0, 1.0 / 6.0, 1e-6),
        (6, 1.0, 0, 0.0, 5.0, 0.0, 0.0), (9, 0.5, 0.5, 0.5, 0.6, 0.5, 0.0), (10, 0.5, 0.5, -0.3, 0.7, 0.7, 0.0),
        (9, 1.0, 1.0, 0.0, 0.0, -0.2, 1e-6), (0, 0, 0, 1.0, 2.0, np.inf, 0.0), (1, 0, 0, 1.0, 2.0, 2.0, 0.0),
        (2, 0, 0, 1.0, 2.0, 1.0, 0.0), (9, 0.5, 0.5, np.inf, 0.3, 0.3, 0.0), (10, 0.5, 0.5, np.inf, -1.0, np.inf, 0.0),
        (11, 0.5, 0.5, 0.4, np.inf, 0.4, 0.0), (11, 0.5, 0.5, np.inf, 0.4, np.inf, 0.0),
        (7, 0.5, 0.5, np.inf, np.inf, np.inf, 0.0),
    ]
    lib = ref_lib()
    prim_ref = np.array([lib.ref_eval_primitive_raw(k, ptr(p), *[C.c_float(v) for v in pt])
                         for k, p, pt, _, _ in rows], np.float32)
    op_ref = []
    for code, k, d, f0, f1, _, _ in ops:
        kd = np.array([k, d], np.float32)
        op_ref.append(lib.ref_eval_operator_raw(code, ptr(kd), C.c_float(f0), C.c_float(f1)))
    np.savez_compressed(
        os.path.join(HERE, "field_known_answers.npz"),
        prim_kind=np.array([r[0] for r in rows], np.uint32), prim_params=np.stack([r[1] for r in rows]),
        prim_point=np.array([r[2] for r in rows], np.float32), prim_expected=np.array([r[3] for r in rows], np.float64),
        prim_tol=np.array([r[4] for r in rows], np.float64), prim_ref=prim_ref,
        op_code=np.array([o[0] for o in ops], np.uint32), op_kd=np.array([[o[1], o[2]] for o in ops], np.float32),
        op_f=np.array([[o[3], o[4]] for o in ops], np.float32), op_expected=np.array([o[5] for o in ops], np.float64),
        op_tol=np.array([o[6] for o in ops], np.float64), op_ref=np.array(op_ref, np.float32))


def scene_fixture(name, w, h):
    cfg = RenderConfig()
    r = RefScene(name, 0, w, h)
    vois = r.vois(cfg.hitEpsilon)
    off, frags, _ = r.rasterize(vois)
    g, st, _ = r.render_tiles(cfg, off, frags, threads=1, normals=True)
    extra = {}
    if name == "csg":
        go, so = r.oracle(cfg, threads=1)
        extra = dict(oracle_hit=go.hit, oracle_depth=go.depth, oracle_evalCount=go.evalCount,
                     oracle_stats=np.array([so.fieldEvals, so.retainedNodeVisits, so.primitiveEvals], np.uint64))
    np.savez_compressed(
        os.path.join(HERE, f"scene_{name.replace(':', '_')}.npz"), name=name, width=w, height=h,
        roi=r.roi(), vois=vois.view(np.uint8), offsets=off, frags=frags.view(np.uint8), hit=g.hit, depth=g.depth,
        evalCount=g.evalCount, normal=g.normal, tileMaxOverlap=g.tileMaxOverlap, tileCacheBytes=g.tileCacheBytes,
        tileError=g.tileError,
        stats=np.array([st.fieldEvals, st.retainedNodeVisits, st.primitiveEvals, st.treeNodeCount, st.maxOverlap,
                        st.maxCacheBytes], np.uint64), **extra)
    print(f"{name}: {len(frags)} fragments, {int(g.hit.sum())} hits")


if __name__ == "__main__":
    field_known_answers()
    for n, w, h in GOLDEN_SCENES:
        scene_fixture(n, w, h)
