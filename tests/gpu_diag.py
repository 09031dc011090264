"""GPU diagnostic report (run on a B200 box): parity of every stage against
the CPU reference plus rough timings.  Not a pytest module; prints a report.

    python tests/gpu_diag.py [scene ...]
"""
from __future__ import annotations

import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle_bridge import RefScene, compare_gbuffers  # noqa: E402
from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32) if a.dtype == np.float32 else a


def diff_count(a, b):
    return int(np.count_nonzero(bits(a) != bits(b)))


def section(title):
    print("\n==== " + title, flush=True)


def run_ref_unit_tests():
    section("reference unit tests against libblobtree_b200.so")
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests_b200")
    if not os.path.exists(exe):
        print("missing", exe)
        return
    t = time.time()
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(p.stdout[-2000:])
    print(p.stderr[-4000:])
    print(f"rc={p.returncode} {time.time() - t:.1f}s")


def scene_report(name, seed=0):
    section(f"scene {name}")
    cfg = RenderConfig()
    s = Scene.build(name, seed)
    r = RefScene(name, seed)
    rd = Renderer(0)
    rd.upload(s)
    cam = s.device_camera
    # (a)
    roi_g = rd.propagate_roi()
    roi_r = r.roi()
    print("roi diff", diff_count(roi_g, roi_r), "of", len(roi_r))
    v_g = rd.build_volumes_of_interest(cfg.hitEpsilon)
    v_r = r.vois(cfg.hitEpsilon)
    print("voi bytes diff", int(np.count_nonzero(v_g.view(np.uint8) != v_r.view(np.uint8))), "vois", len(v_r))
    # (b)
    t0 = time.perf_counter()
    off_g, fr_g = rd.rasterize_volumes(cam)
    t_gpu_ab = time.perf_counter() - t0
    off_r, fr_r, ms_ref_ab = r.rasterize(v_r)
    same_off = bool((off_g == off_r).all())
    same_fr = len(fr_g) == len(fr_r) and bool((fr_g.view(np.uint8) == fr_r.view(np.uint8)).all())
    print(f"abuffer fragments gpu={len(fr_g)} ref={len(fr_r)} offsets_equal={same_off} frags_bitexact={same_fr} "
          f"ref_ms={ms_ref_ab:.1f} gpu_call_ms={t_gpu_ab * 1e3:.1f}")
    if not same_off:
        cg = np.diff(off_g.astype(np.int64))
        cr = np.diff(off_r.astype(np.int64))
        bad = np.nonzero(cg != cr)[0]
        print("  tiles with count diff:", len(bad), "first", bad[:10], cg[bad[:10]], cr[bad[:10]])
    # (c) exact, on the GPU A-buffer (identical to the reference's if bit-exact above)
    rd.reset_stats()
    t0 = time.perf_counter()
    rd.render_tiles(cam, cfg, exact=True)
    rd.compute_normals(cam, 0, exact=True)
    rd.sync()
    t_gpu_tr = time.perf_counter() - t0
    g = rd.download_gbuffer()
    st = rd.stats()
    gr, str_, ms = r.render_tiles(cfg, off_r, fr_r, threads=0, normals=True)
    print(f"exact trace: hit diff {diff_count(g.hit, gr.hit)} depth diff {diff_count(g.depth, gr.depth)} "
          f"evals diff {diff_count(g.evalCount, gr.evalCount)} normal diff {diff_count(g.normal, gr.normal)} "
          f"tmo diff {diff_count(g.tileMaxOverlap, gr.tileMaxOverlap)} tcb diff "
          f"{diff_count(g.tileCacheBytes, gr.tileCacheBytes)} terr diff {diff_count(g.tileError, gr.tileError)}")
    print(f"  stats gpu fe={st.fieldEvals} rnv={st.retainedNodeVisits} pe={st.primitiveEvals} mo={st.maxOverlap} "
          f"mc={st.maxCacheBytes} flops={st.fieldFlops} fallbacks={st.normalFallbacks} errors={st.tileErrors}")
    print(f"  stats ref fe={str_.fieldEvals} rnv={str_.retainedNodeVisits} pe={str_.primitiveEvals} "
          f"mo={str_.maxOverlap} mc={str_.maxCacheBytes}")
    print(f"  hits={int(gr.hit.sum())} of {len(gr.hit)}; ref trace ms={ms[0]:.1f} normals ms={ms[1]:.1f}; "
          f"gpu call ms={t_gpu_tr * 1e3:.1f}")
    if diff_count(g.hit, gr.hit):
        bad = np.nonzero(g.hit != gr.hit)[0][:10]
        print("  first hit mismatches", bad, g.hit[bad], gr.hit[bad], g.evalCount[bad], gr.evalCount[bad])
    # fast mode
    rd.render_tiles(cam, cfg, exact=False)
    rd.compute_normals(cam, 0, exact=False)
    gf = rd.download_gbuffer()
    rep = compare_gbuffers(gf, gr, 2 * cfg.minStep)
    both = (gf.hit == 1) & (gr.hit == 1)
    dots = (gf.normal[both] * gr.normal[both]).sum(1) if both.any() else np.ones(1)
    print(f"fast trace vs ref: {rep}  normal dot>=0.999: {float((dots >= 0.999).mean()):.5f}")
    # frame path + timing
    for graph in (False, True):
        rd.render_frame(cam, cfg, exact=False, graph=graph)
        rd.sync()
        n = 20
        t0 = time.perf_counter()
        for _ in range(n):
            rd.render_frame(cam, cfg, exact=False, graph=graph)
        rd.sync()
        dt = (time.perf_counter() - t0) / n
        print(f"render_frame graph={graph}: {dt * 1e3:.3f} ms/frame wall  ({s.width * s.height / dt / 1e6:.0f} Mrays/s)")
    gff = rd.download_gbuffer()
    print("frame vs separate-stage fast hit diff", diff_count(gff.hit, gf.hit), "depth diff",
          diff_count(gff.depth, gf.depth))
    rd.profile(True)
    rd.rasterize_volumes(cam)
    rd.render_tiles(cam, cfg, exact=False)
    rd.compute_normals(cam, 0, exact=False)
    ms4, n4 = rd.profile_read()
    print("per-stage device ms [roi/voi, abuffer, trace, normals]:", ms4, n4)
    rd.profile(False)
    rd.close()


def main():
    names = sys.argv[1:] or ["sphere", "csg", "comb_error", "random:24", "C1", "C2", "C3", "C5"]
    import subprocess as sp
    print(sp.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm,driver_version", "--format=csv"],
                 capture_output=True, text=True).stdout)
    run_ref_unit_tests()
    for n in names:
        try:
            scene_report(n)
        except Exception as e:  # keep going
            import traceback
            traceback.print_exc()
            print("FAILED", n, e)


if __name__ == "__main__":
    main()
