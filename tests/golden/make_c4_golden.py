"""Generate tests/golden/c4_reference.npz from the UNMODIFIED reference
(oracle/_ref/libbt_ref.so, built from /root/reference/proj/src).

    python tests/golden/make_c4_golden.py

C4: 10,000 primitives at 3840x2160, 129,600 tiles.
The reference's rasterize_volumes is single-threaded by design
(abuffer.cpp:175-225) and takes ~30 s here, so the GPU box -- which has no
/root/reference -- checks against this fixture instead of a live run:

* the reference's CSR A-buffer: the per-tile offsets themselves, and SHA-256
  digests of the Fragment{word, zEntry, zExit} array (bit-exact membership,
  order and depths), whole and per tile row (a failing GPU run reports the
  rows that differ; the 1.15 M fragments themselves would be 14 MB);
* SHA-256 digests of every plane of the reference pipeline's G-buffer
  (render_tiles, tracer.cpp:141-236, + compute_normals, :296-350, the
  composition of test_tracer.cpp:25-31), whole and per tile row, and its
  RenderStats.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle_bridge import RefScene  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig  # noqa: E402

PLANES = ("hit", "depth", "normal", "evalCount", "tileMaxOverlap", "tileCacheBytes", "tileError")


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def row_digests(a: np.ndarray, rows: int) -> np.ndarray:
    """digest of each of `rows` equal horizontal bands of a per-pixel or per-tile plane"""
    a = np.ascontiguousarray(a)
    per = len(a) // rows
    return np.array([digest(a[i * per:(i + 1) * per]) for i in range(rows)])


def frag_row_digests(off: np.ndarray, frags: np.ndarray, tiles_x: int, tiles_y: int) -> np.ndarray:
    return np.array([digest(frags[off[y * tiles_x]:off[(y + 1) * tiles_x]]) for y in range(tiles_y)])


def main(name: str = "C4", out: str = os.path.join(HERE, "c4_reference.npz")) -> None:
    cfg = RenderConfig()
    r = RefScene(name)
    t0 = time.time()
    vois = r.vois(cfg.hitEpsilon)
    off, frags, ms_ab = r.rasterize(vois)
    g, st, _ = r.render_tiles(cfg, off, frags, threads=0, normals=True)
    print(f"{name}: {len(frags)} fragments, rasterize {ms_ab / 1e3:.1f} s, total {time.time() - t0:.1f} s")
    stats = np.array([st.fieldEvals, st.retainedNodeVisits, st.primitiveEvals, st.treeNodeCount, st.maxOverlap,
                      st.maxCacheBytes], np.uint64)
    tx, ty = r.tiles
    np.savez_compressed(
        out, scene=np.array(name), width=np.int32(r.width), height=np.int32(r.height),
        offsets=off, frag_count=np.uint64(len(frags)), frag_digest=np.array(digest(frags)),
        frag_row_digests=frag_row_digests(off, frags, tx, ty), voi_digest=np.array(digest(vois)),
        plane_names=np.array(PLANES), plane_digests=np.array([digest(getattr(g, p)) for p in PLANES]),
        plane_row_digests=np.stack([row_digests(getattr(g, p), ty) for p in PLANES]), stats=stats)
    print(f"wrote {out} ({os.path.getsize(out) / 1e6:.1f} MB)")


if __name__ == "__main__":
    main(*sys.argv[1:])
