#!/usr/bin/env python
"""bench.py -- synchronized tracing of a 1,000-primitive blobtree at 1080p.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one frame of the reference's per-frame pipeline on the C3 workload
(SURVEY.md appendix C): per-frame primitive-parameter update (all 1,000
primitives perturbed) -> (a) ROI + VOIs -> (b) 8x8-tile A-buffer -> (c)
synchronized sphere tracing -> normals, replayed from one CUDA graph.

* value       Mrays/s = W*H / device time per frame (CUDA events on the
              stream the kernels run on; L2 flushed between frames by a
              256 MiB write that is not timed); inputs resident in HBM.
* e2e         the same through the public C-ABI with HOST buffers: pinned
              H2D of the frame's parameter deltas and D2H of the whole
              G-buffer (hit, depth, normal, evalCount, tile planes) per step.
* roofline    the field-evaluation kernel (k_march) against the measured FP32
              (FFMA) peak of the box: algorithmic flops per frame (SURVEY.md
              appendix B, counted on the device) / the kernel's CUDA-event time.
* cpu_baseline the unmodified reference (oracle/_ref) timed on this host's
              cores on one C3 frame.
--impl reference times that reference CPU path per step instead.
Multi-GPU (torchrun): the frame's tile rows are split over ranks (strong
scaling); each rank traces its rows straight into rank 0's G-buffer over
peer memory (fused gather, CUDA IPC; NCCL gather as the fallback) and shades
its own rows' normals there.  Beside the C3 headline every run also times
the C4 scaling config (scaling_c4).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mrays/s and ms/frame at 1080p vs primitive count; % FP32 peak (field eval)"
WORKLOAD = ("C3: synthetic blobtree, 1,000 primitives (250 compact-union cells x 4, sharp-union comb), "
            "1920x1080, all primitive parameters perturbed every frame")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--exact", action="store_true", help="IEEE-exact kernels instead of FMA field evaluation")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--split", default="cost", choices=["cost", "even"],
                    help="multi-GPU tile-row split: balanced by each row's march cost, or even row counts")
    return ap.parse_args()


# ---------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------- shared config

CONFIG_SIZES = {"C1": (10, 512, 512), "C2": (142, 1920, 1080), "C3": (1000, 1920, 1080), "C4": (10000, 3840, 2160),
                "C5": (4000, 1920, 1080)}


def bench_config(config: str, arm: dict) -> dict:
    """The `config` object of both arms: the same keys, the workload keys with
    the same values; `arm` fills what differs by nature (field arithmetic,
    L2 handling, parallelism)."""
    prims, w, h = CONFIG_SIZES.get(config, (None, None, None))
    out = {"workload": WORKLOAD if config == "C3" else config, "primitives": prims,
           "resolution": f"{w}x{h}" if w else None, "rays_per_frame": w * h if w else None,
           "field_eval": None, "l2": None, "parallelism": None, "graph": None}
    out.update(arm)
    return out


def host_cpu() -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


# ---------------------------------------------------------------------------- reference arm

def cpu_frame_reference(config: str, frames: int, threads: int, median: bool = False):
    """Time the unmodified reference library (oracle/_ref) on `frames`
    perturbed frames.  Returns (rays, wall seconds per frame, per-stage ms:
    the mean over all frames, or with median=True the median over all but the
    first, warm-up frame)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bridge import RefScene, ref_available  # CPU checker: bench's CPU legs only
    from paper_2304_09673_b200.pipeline import RenderConfig
    if not ref_available():
        return None
    cfg = RenderConfig()
    r = RefScene(config)
    times, stages = [], []
    for f in range(frames):
        r.perturb(f)
        t0 = time.perf_counter()
        _, _, ms, _ = r.frame(cfg, threads)
        times.append(time.perf_counter() - t0)
        stages.append(ms)
    if median:
        return r.width * r.height, times, np.median(np.asarray(stages[1:]), axis=0)
    return r.width * r.height, times, np.mean(stages, axis=0)


def run_reference(args, rank: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    out = cpu_frame_reference(args.config, args.warmup + args.steps, threads)
    if out is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbt_ref.so not built (needs "
                                                               "/root/reference at build time)"}))
        return
    rays, times, stages = out
    timed = times[args.warmup:]
    ms = 1e3 * float(np.mean(timed))
    value = rays / (ms * 1e-3) / 1e6
    sample = (f"{len(timed)} full {args.config} frames: propagate_roi+build_volumes_of_interest, rasterize_volumes "
              f"(single-threaded by design), render_tiles ({threads} threads), compute_normals; mean stage ms "
              f"{[round(float(s), 2) for s in stages]}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "Mrays/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.config, {
            "field_eval": "ieee (the reference's own CPU code, unmodified)",
            "l2": "n/a (CPU path; each frame re-reads the whole scene from host memory)",
            "parallelism": f"{threads} host threads (render_tiles, oracle_render); rasterize_volumes single-threaded",
            "graph": "n/a"}),
        "host_cpu": host_cpu(),
        "cpu_baseline": {"value": round(value, 3), "unit": "Mrays/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- B200 arm

class ShardedFrames:
    """One rank's share of the frame sequence of a config: the scene, its
    renderer on this rank's stream, the per-frame parameter deltas resident
    in HBM, the rank's tile rows, and the exchange with the other ranks.

    Multi-GPU exchange.  Preferred: the fused gather -- rank 0 exports its
    G-buffer planes (CUDA IPC), the other ranks import them, so every march
    writes its rows straight into rank 0's G-buffer over NVLink while it
    runs; a one-element all-reduce on the stream then orders every rank's
    normals (its own rows, the one-row depth halo read from rank 0's planes,
    written into rank 0's normal plane) after every rank's march, and a
    second one orders the next frame's peer writes after every rank's
    normals.  Fallback: NCCL gather of the rows, normals on rank 0."""

    def __init__(self, config, args, rank, world, dev, stream, frames):
        import ctypes as C

        import torch

        from paper_2304_09673_b200 import _capi as capi
        from paper_2304_09673_b200.distributed import tile_row_ranges
        from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene
        self.rank, self.world, self.dev = rank, world, dev
        self.scene = Scene.build(config)
        self.rd = Renderer(dev.index)
        self.rd.set_stream(stream.cuda_stream)
        self.rd.upload(self.scene)
        self.lib = self.rd.lib
        self.cam = self.scene.device_camera
        self.cfg = RenderConfig()
        self.exact = bool(args.exact)
        self.W, self.H = self.scene.width, self.scene.height
        tiles_x, tiles_y = self.scene.tiles
        # strong scaling: contiguous tile-row ranges per rank, balanced by the
        # march cost of each row (the field evaluations of one full frame,
        # computed on rank 0 and broadcast) -- the middle rows of a frame
        # carry most of the surface; an even split leaves the edge ranks idle
        self.rows = tile_row_ranges(tiles_y, world)
        if world > 1 and getattr(args, "split", "cost") == "cost":
            import torch.distributed as dist

            from paper_2304_09673_b200.distributed import row_costs
            obj = [None]
            if rank == 0:
                self.rd.render_frame(self.cam, self.cfg, exact=self.exact, graph=False)
                g = self.rd.download_gbuffer()
                obj = [tile_row_ranges(tiles_y, world, row_costs(g.evalCount, self.W, self.H)).tolist()]
            dist.broadcast_object_list(obj, src=0)
            self.rows = np.asarray(obj[0], np.int64)
        self.tile0, self.tile1 = int(self.rows[rank] * tiles_x), int(self.rows[rank + 1] * tiles_x)
        if world == 1:
            self.tile0, self.tile1 = 0, 0
        # all frames' parameter deltas resident in HBM before timing
        self.host_frames = [self.scene.perturb(f) for f in range(frames)]
        self.nprim = len(self.scene.prims)
        self.d_words = [torch.from_numpy(w.view(np.int32)).to(dev) for w, _, _ in self.host_frames]
        self.d_params = [torch.from_numpy(p).to(dev) for _, p, _ in self.host_frames]
        self.d_counts = [torch.from_numpy(c.view(np.int32)).to(dev) for _, _, c in self.host_frames]
        self.planes = {}
        self.fused = False
        if world > 1:
            import torch.distributed as dist
            self.rd.render_frame(self.cam, self.cfg, exact=self.exact, graph=False, tile0=self.tile0,
                                 tile1=self.tile1, normals=False)
            torch.cuda.synchronize(dev)
            ok = 1
            h = capi.bt_ipc_handles()
            if rank == 0 and self.lib.bt_gbuffer_export(self.rd.ctx, C.byref(h)) != 0:
                ok = 0
            obj = [bytes(h), ok]
            dist.broadcast_object_list(obj, src=0)
            if obj[1] and rank != 0:
                C.memmove(C.addressof(h), obj[0], C.sizeof(h))
                ok = 1 if self.lib.bt_gbuffer_import(self.rd.ctx, C.byref(h)) == 0 else 0
            flag = torch.tensor([ok if obj[1] else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            self.fused = bool(flag.item())
            if not self.fused and rank != 0:
                self.lib.bt_gbuffer_import_release(self.rd.ctx)
            self.done = torch.zeros(1, dtype=torch.int32, device=dev)

    def render(self, f):
        """frame f up to a complete G-buffer on rank 0 (device-resident deltas)"""
        rd, world = self.rd, self.world
        rd.update_params_device(self.d_words[f].data_ptr(), self.d_params[f].data_ptr(), self.d_counts[f].data_ptr(),
                                self.nprim)
        self.render_rows()

    def render_rows(self):
        from paper_2304_09673_b200.distributed import gather_rows, gbuffer_planes
        rd, world = self.rd, self.world
        rd.render_frame(self.cam, self.cfg, exact=self.exact, graph=True, tile0=self.tile0, tile1=self.tile1,
                        normals=(world == 1))
        if world == 1:
            return
        import torch.distributed as dist
        if self.fused:
            dist.all_reduce(self.done)  # stream-ordered: every rank's march has written its rows
            rd.compute_normals_rows(self.cam, self.tile0, self.tile1, self.cfg.normalsMode, self.exact)
            dist.all_reduce(self.done)  # every rank's normals are in: the frame is complete on rank 0
        else:
            # this rank's rows of hit/depth/evalCount -> rank 0 (NCCL), normals on rank 0
            if not self.planes:
                self.planes.update(gbuffer_planes(rd.gbuffer_device(), self.dev))
            gather_rows(self.planes, self.rows, self.rank, world, self.W, self.H)
            if self.rank == 0:
                rd.compute_normals(self.cam, self.cfg.normalsMode, self.exact)

    def release(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
            if self.fused and self.rank != 0:
                self.lib.bt_gbuffer_import_release(self.rd.ctx)
            dist.barrier()
        self.rd.close()


def device_ms(fr, args, stream, flush, f0=0):
    """CUDA-event ms per frame over args.steps frames after args.warmup
    untimed ones (L2 flushed between frames, untimed), max over ranks."""
    import torch
    dev = fr.dev
    for f in range(args.warmup):
        fr.render(f0 + f)
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if fr.world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        fr.render(f0 + args.warmup + i)
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    if fr.world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def run_b200(args, rank: int, world: int, local_rank: int):
    import ctypes as C

    import torch

    from paper_2304_09673_b200 import _capi as capi

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # a real (non-NULL) stream shared by torch and the library: the events
    # below record on the stream the kernels actually run on
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    lib = capi.load()

    nframes = args.warmup + args.steps
    fr = ShardedFrames(args.config, args, rank, world, dev, stream, nframes)
    scene, rd, cam, cfg, exact = fr.scene, fr.rd, fr.cam, fr.cfg, fr.exact
    W, H = fr.W, fr.H
    tiles_x, tiles_y = scene.tiles
    tile0, tile1, rows, fused, planes = fr.tile0, fr.tile1, fr.rows, fr.fused, fr.planes
    host_frames, nprim = fr.host_frames, fr.nprim
    d_words, d_params, d_counts = fr.d_words, fr.d_params, fr.d_counts
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(f):
        fr.render(f)

    for f in range(args.warmup):
        step(f)
    torch.cuda.synchronize(dev)

    # ------------------------------------------------------------------ timed region
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    rd.reset_stats()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local_rank) as clocks:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step(args.warmup + i)
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    # a graph replay that outgrew a capacity only flags it (the frame is
    # emptied, never written out of bounds): bt_stats_download raises
    # BT_ENOMEM then, and a flagged frame must not be reported as a speed
    st_timed = rd.stats()
    assert st_timed.tileErrors == 0, f"{st_timed.tileErrors} tile errors in the timed frames"
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clock = clocks.summary()
    kernels, nodes = C.c_uint32(), C.c_uint32()
    capi.check(lib.bt_graph_kernel_count(rd.ctx, C.byref(kernels), C.byref(nodes)), "bt_graph_kernel_count")
    launches = args.steps * (kernels.value + 1)  # graph kernels + the parameter-update kernel
    value = W * H / (ms * 1e-3) / 1e6

    e2e_multi = None
    if world > 1:
        e2e_multi = e2e_pass_multi(fr, args)
    scaling = None
    if not args.no_sweep:  # the C4 scaling curve beside the headline, at every N
        scaling = scaling_block("C4", args, rank, world, dev, stream, flush)
    if rank != 0:
        return
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (procedural scene, fixed seed)",
        "config": bench_config(args.config, {
            "field_eval": "ieee-exact" if exact else "fma-contracted (tolerance path)",
            "l2": "flushed between timed frames (256 MiB device write, untimed)",
            "parallelism": (f"tile rows over {world} GPU(s) ({args.split}-balanced split), "
                            f"{'fused gather + per-rank normals (IPC peer memory)' if fused else 'NCCL gather'}")
                           if world > 1 else "1 GPU",
            "graph": f"{kernels.value} kernels / {nodes.value} nodes per frame"}),
        "gpu_launches": launches,
        "clocks": {k: clock[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
    }
    if scaling is not None:
        result["scaling_c4"] = scaling

    # ------------------------------------------------------------------ per-stage + roofline (untimed pass)
    stage_ms, flops_per_frame, st = stage_breakdown(rd, cam, cfg, exact, d_words, d_params, d_counts, nprim)
    peak = C.c_float()
    capi.check(lib.bt_fp32_peak(local_rank, C.byref(peak), None), "bt_fp32_peak")
    march_ms = stage_ms["trace_march"]
    achieved = flops_per_frame / (march_ms * 1e-3) / 1e12
    result["stages_ms"] = {k: round(v, 4) for k, v in stage_ms.items()}
    result["roofline"] = {
        "kernel": "k_march (synchronized per-tile sphere tracing + field evaluation)",
        "kernel_ms": round(march_ms, 4),
        "bound": "fp32", "achieved": round(achieved, 3), "peak": round(peak.value, 2), "unit": "TFLOP/s",
        "frac": round(achieved / peak.value, 4), "traffic": None,
        "peak_source": "measured FFMA microbenchmark on this box (bt_fp32_peak); MEASURED_PEAKS.json has no FP32 figure",
        "work": f"{flops_per_frame / 1e9:.3f} GFLOP/frame algorithmic (SURVEY.md appendix B), "
                f"{st.fieldEvals} field evals/frame",
    }
    traffic_path = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(traffic_path):  # dram read+write bytes of one k_march launch (ncu --set full, committed)
        trs = json.load(open(traffic_path))
        tr = trs.get(f"k_march@{args.config.lower()}")
        if tr:
            result["roofline"]["traffic"] = tr["dram_bytes_per_launch"]
            result["roofline"]["traffic_source"] = tr["source"]
            if "fp32_executed_flops" in tr:
                # the SASS FP32 work actually executed (2 FFMA + FADD + FMUL, ncu of one launch of this config) over the same
                # live kernel time: appendix B credits the reference's formulas (e.g. 33 flop of quaternion
                # transform that the fast path executes as 9 FFMA), the executed count does not
                ex = tr["fp32_executed_flops"] / (march_ms * 1e-3) / 1e12
                result["roofline"]["executed"] = {"achieved": round(ex, 3), "frac": round(ex / peak.value, 4),
                                                  "flops_per_launch": tr["fp32_executed_flops"],
                                                  "source": tr["source"]}
    # (b) A-buffer build, HBM-bound by SURVEY.md 8(d): algorithmic bytes =
    # V x 64 (volumes read) + T x 8 (CSR offset + count) + F x 12 (fragments written)
    hbm = None
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        hbm = json.load(open(peaks_path)).get("hbm_gbs")
    ab_bytes = nprim * 64 + tiles_x * tiles_y * 8 + st.fragments * 12
    ab_gbs = ab_bytes / (stage_ms["abuffer"] * 1e-3) / 1e9
    result["abuffer_roofline"] = {
        "kernels": "k_camera, k_pairs, k_scan, k_sb_scatter, k_tile_raster", "bound": "hbm",
        "achieved": round(ab_gbs, 2), "peak": hbm, "unit": "GB/s",
        "frac": round(ab_gbs / hbm, 5) if hbm else None, "algorithmic_bytes": ab_bytes,
        "note": "bound by the exact IEEE ray tests (instruction issue), not HBM: the algorithmic traffic is ~2 MB per frame",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (driver-written)"}
    result["frame_stats"] = {"fieldEvals": st.fieldEvals, "warpSteps": st.warpSteps,
                             "laneUtilisation": round(st.fieldEvals / max(1, 32 * st.warpSteps), 4),
                             "fragments": st.fragments,
                             "candidatePairs": st.candidatePairs, "maxOverlap": st.maxOverlap,
                             "normalFallbacks": st.normalFallbacks, "tileErrors": st.tileErrors}

    # ------------------------------------------------------------------ e2e through the C-ABI with host buffers
    if world == 1:
        result["e2e"] = e2e_pass(rd, scene, cam, cfg, exact, host_frames, args)
    elif e2e_multi is not None:
        result["e2e"] = e2e_multi

    # ------------------------------------------------------------------ CPU reference beside it
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        out = cpu_frame_reference(args.config, 6, threads, median=True)
        if out is not None:
            rays, times, stages = out
            med = float(np.median(times[1:]))
            v = rays / med / 1e6
            names = ("roi_voi", "rasterize_volumes", "render_tiles", "compute_normals")
            result["cpu_baseline"] = {
                "value": round(v, 3), "unit": "Mrays/s", "cores": threads, "kind": "reference",
                "host_cpu": host_cpu(), "ms_per_frame": round(med * 1e3, 2),
                "stages_ms_median": {n: round(float(x), 2) for n, x in zip(names, stages)},
                "sample": f"6 perturbed {args.config} frames through the unmodified reference (oracle/_ref), the "
                          f"first a warm-up, per-stage median of the other 5: rasterize_volumes single-threaded by "
                          f"design, render_tiles and compute_normals on {threads} threads; the reference's "
                          f"steady_clock stage timers"}
    if not args.no_sweep and world == 1:
        result["sweep_ms_per_frame"] = sweep(rd, exact)
        result["frames_in_flight"] = frames_in_flight(scene, cam, cfg, exact, d_words, d_params, d_counts, nprim)
    print(json.dumps(result), flush=True)


def stage_breakdown(rd, cam, cfg, exact, d_words, d_params, d_counts, nprim, frames: int = 5):
    """Eager pass with CUDA events around each stage (bt_profile_*)."""
    import ctypes as C

    from paper_2304_09673_b200 import _capi as capi
    lib = rd.lib
    c = cfg.to_c()
    rd.profile(True)
    st = None
    flops = []
    for i in range(frames):
        f = i % len(d_words)  # short runs (--steps 2 --warmup 1) cycle the prepared frames
        rd.update_params_device(d_words[f].data_ptr(), d_params[f].data_ptr(), d_counts[f].data_ptr(), nprim)
        rd.reset_stats()
        capi.check(lib.bt_roi(rd.ctx, None, 0), "bt_roi")
        capi.check(lib.bt_voi_build(rd.ctx, C.c_float(cfg.hitEpsilon)), "bt_voi_build")
        capi.check(lib.bt_abuffer_build(rd.ctx, C.byref(cam), 0, 0), "bt_abuffer_build")
        capi.check(lib.bt_trace(rd.ctx, C.byref(cam), C.byref(c), 0, 0, int(exact)), "bt_trace")
        capi.check(lib.bt_normals(rd.ctx, C.byref(cam), cfg.normalsMode, int(exact)), "bt_normals")
        st = rd.stats()
        flops.append(st.fieldFlops)
    ms, n = rd.profile_read_ex()
    rd.profile(False)
    names = ["roi_voi", "abuffer", "trace", "normals", "trace_views", "trace_march"]
    stage = {names[i]: float(ms[i]) / max(int(n[i]), 1) for i in range(6)}
    stage["roi_voi"] *= 2  # roi and voi are two profiled calls per frame
    return stage, float(np.mean(flops)), st


def e2e_pass(rd, scene, cam, cfg, exact, host_frames, args) -> dict:
    """Through the C-ABI with host buffers, wall clock: per step the pinned H2D
    of the frame's parameter deltas, the frame, and the D2H of the whole
    G-buffer into pinned host memory.  Streaming (the headline): the download
    is bt_gbuffer_download_async -- snapshot on the device, copy on the
    context's copy stream into one of two host buffer sets -- so frame N's
    transfer overlaps frame N+1's render; every frame still reaches the host
    inside the timed region (bt_download_wait at the end).  Also reported:
    the fully synchronous variant (bt_gbuffer_download, frame by frame)."""
    import torch
    W, H = scene.width, scene.height
    tx, ty = scene.tiles
    n = len(scene.prims)
    pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
    frames = [(pin(w.view(np.int32)), pin(p), pin(c.view(np.int32))) for w, p, c in host_frames]
    planes = ("hit", "depth", "normal", "evalCount", "tmo", "tcb", "terr")

    lib = rd.lib
    import ctypes as C
    from paper_2304_09673_b200 import _capi as capi
    off = (C.c_size_t * 7)()
    total = C.c_size_t()
    capi.check(lib.bt_gbuffer_layout(rd.ctx, off, C.byref(total)), "bt_gbuffer_layout")

    def host_set():
        # one pinned slab per set, planes at bt_gbuffer_layout's offsets: the
        # download merges them into two copies
        slab = torch.empty(total.value, dtype=torch.uint8).pin_memory()
        spec = (("hit", W * H, torch.uint8), ("depth", W * H, torch.float32), ("normal", W * H * 3, torch.float32),
                ("evalCount", W * H, torch.int32), ("tmo", tx * ty, torch.int32), ("tcb", tx * ty, torch.int32),
                ("terr", tx * ty, torch.uint8))
        out = {k: slab[off[i]:off[i] + n * torch.empty(0, dtype=d).element_size()].view(d)
               for i, (k, n, d) in enumerate(spec)}
        out["_slab"] = slab
        return out
    outs = [host_set(), host_set()]

    def step(f, stream_dl):
        w, p, c = frames[f]
        capi.check(lib.bt_params_update(rd.ctx, C.c_void_p(w.data_ptr()), C.c_void_p(p.data_ptr()),
                                        C.c_void_p(c.data_ptr()), n, 17), "bt_params_update")
        rd.render_frame(cam, cfg, exact=exact, graph=True)
        out = outs[f % 2]
        args_ = [C.c_void_p(out[k].data_ptr()) for k in planes]
        if stream_dl:
            capi.check(lib.bt_gbuffer_download_async_slab(rd.ctx, C.c_void_p(out["_slab"].data_ptr())),
                       "bt_gbuffer_download_async_slab")
        else:
            capi.check(lib.bt_gbuffer_download(rd.ctx, *args_), "bt_gbuffer_download")

    def timed(stream_dl):
        for f in range(args.warmup):
            step(f, stream_dl)
        capi.check(lib.bt_sync(rd.ctx), "bt_sync")
        t0 = time.perf_counter()
        for i in range(args.steps):
            step(args.warmup + i, stream_dl)
        capi.check(lib.bt_download_wait(rd.ctx), "bt_download_wait")
        capi.check(lib.bt_sync(rd.ctx), "bt_sync")
        return (time.perf_counter() - t0) / args.steps

    dt_sync = timed(False)
    dt = timed(True)
    # the last frame's G-buffer on the host equals the device's
    g = rd.download_gbuffer()
    last = outs[(args.warmup + args.steps - 1) % 2]
    assert np.array_equal(last["depth"].numpy(), g.depth.reshape(-1)), "streamed G-buffer differs from the device's"
    h2d = n * (4 + 17 * 4 + 4)
    d2h = W * H * (1 + 4 + 12 + 4) + tx * ty * (4 + 4 + 1)
    return {"value": round(W * H / dt / 1e6, 2), "unit": "Mrays/s", "ms_per_step": round(dt * 1e3, 4),
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "bt_params_update (pinned host) -> bt_render_frame -> bt_gbuffer_download_async_slab (one pinned host slab, "
                    "copy stream; frame N's D2H overlaps frame N+1's render), wall clock",
            "sync_variant": {"value": round(W * H / dt_sync / 1e6, 2), "ms_per_step": round(dt_sync * 1e3, 4),
                             "path": "same with the blocking bt_gbuffer_download per frame"}}


def e2e_pass_multi(fr, args) -> dict | None:
    """N GPUs end to end, wall clock, max over ranks: per step every rank
    uploads the frame's parameter deltas from pinned host memory, traces its
    tile rows into rank 0's G-buffer and shades their normals there (fused
    gather; or the NCCL gather + normals on rank 0); rank 0 streams the whole
    G-buffer into a pinned host slab; every frame is on the host when the
    timed region ends."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2304_09673_b200 import _capi as capi
    rd, lib, rank, world, dev = fr.rd, fr.lib, fr.rank, fr.world, fr.dev
    W, H = fr.W, fr.H
    n = fr.nprim
    pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
    frames = [(pin(w.view(np.int32)), pin(p), pin(c.view(np.int32))) for w, p, c in fr.host_frames]
    slabs = []
    if rank == 0:
        off = (C.c_size_t * 7)()
        total = C.c_size_t()
        capi.check(lib.bt_gbuffer_layout(rd.ctx, off, C.byref(total)), "bt_gbuffer_layout")
        slabs = [torch.empty(total.value, dtype=torch.uint8).pin_memory() for _ in range(2)]

    def step(f, i):
        w, p, c = frames[f]
        capi.check(lib.bt_params_update(rd.ctx, C.c_void_p(w.data_ptr()), C.c_void_p(p.data_ptr()),
                                        C.c_void_p(c.data_ptr()), n, 17), "bt_params_update")
        fr.render_rows()
        if rank == 0:
            capi.check(lib.bt_gbuffer_download_async_slab(rd.ctx, C.c_void_p(slabs[i % 2].data_ptr())),
                       "bt_gbuffer_download_async_slab")
        if fr.fused:  # the snapshot is taken: the next frame's peer writes may land
            dist.all_reduce(fr.done)

    for i in range(args.warmup):
        step(i, i)
    if rank == 0:
        capi.check(lib.bt_download_wait(rd.ctx), "bt_download_wait")
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i, i)
    if rank == 0:
        capi.check(lib.bt_download_wait(rd.ctx), "bt_download_wait")
    torch.cuda.synchronize(dev)
    dt = torch.tensor([(time.perf_counter() - t0) / args.steps], device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    dt = float(dt.item())
    tx, ty = fr.scene.tiles
    return {"value": round(W * H / dt / 1e6, 2), "unit": "Mrays/s", "ms_per_step": round(dt * 1e3, 4),
            "h2d_bytes_per_step": world * n * (4 + 17 * 4 + 4),
            "d2h_bytes_per_step": W * H * (1 + 4 + 12 + 4) + tx * ty * (4 + 4 + 1),
            "path": "every rank: bt_params_update (pinned host) -> bt_render_frame (its tile rows) -> "
                    + ("bt_normals_rows (its rows, into rank 0's planes over peer memory)" if fr.fused else
                       "NCCL gather to rank 0 -> bt_normals on rank 0")
                    + "; rank 0: bt_gbuffer_download_async_slab (pinned host); wall clock, max over ranks"}


def scaling_block(config, args, rank, world, dev, stream, flush) -> dict:
    """The multi-GPU scaling config (C4, 10,000 primitives at
    3840x2160) timed the same way as the headline at this N (device time,
    max over ranks), so the driver's N = 1, 2, 4, 8 runs carry a C4 curve
    beside the C3 one."""
    fr = ShardedFrames(config, args, rank, world, dev, stream, args.warmup + args.steps)
    ms = device_ms(fr, args, stream, flush)
    out = {"config": config, "n_gpus": world, "ms_per_frame": round(ms, 4),
           "Mrays_s": round(fr.W * fr.H / (ms * 1e-3) / 1e6, 1),
           "exchange": ("fused gather + per-rank normals over peer memory" if fr.fused else "NCCL gather")
           if world > 1 else "none"}
    fr.release()
    return out


def eager_stages(r, cam, cfg, exact, frames: int = 3) -> dict:
    """Per-stage device ms of eager frames (CUDA events around each stage)."""
    import ctypes as C

    from paper_2304_09673_b200 import _capi as capi
    lib, c = r.lib, cfg.to_c()
    r.profile(True)
    for _ in range(frames):
        capi.check(lib.bt_roi(r.ctx, None, 0), "bt_roi")
        capi.check(lib.bt_voi_build(r.ctx, C.c_float(cfg.hitEpsilon)), "bt_voi_build")
        capi.check(lib.bt_abuffer_build(r.ctx, C.byref(cam), 0, 0), "bt_abuffer_build")
        capi.check(lib.bt_trace(r.ctx, C.byref(cam), C.byref(c), 0, 0, int(exact)), "bt_trace")
        capi.check(lib.bt_normals(r.ctx, C.byref(cam), cfg.normalsMode, int(exact)), "bt_normals")
    ms, n = r.profile_read_ex()
    r.profile(False)
    names = ["roi_voi", "abuffer", "trace", "normals", "trace_views", "trace_march"]
    out = {names[i]: round(float(ms[i]) / max(int(n[i]), 1), 4) for i in range(6)}
    out["roi_voi"] = round(out["roi_voi"] * 2, 4)
    return out


def frames_in_flight(scene, cam, cfg, exact, d_words, d_params, d_counts, nprim, frames: int = 40) -> dict:
    """Throughput with 2 and 3 frames in flight: as many contexts (each with its
    own tree copy, buffers, CUDA graph and stream) render alternate frames of
    the same perturbed sequence, so one frame's latency-bound stages overlap
    another frame's march.  Reported beside the headline, not as it: the
    headline renders frames back to back, so its ms/frame is also the frame
    latency."""
    import torch

    from paper_2304_09673_b200.pipeline import Renderer
    out = {}
    dev = torch.cuda.current_device()
    for n in (2, 3):
        streams = [torch.cuda.Stream() for _ in range(n)]
        rs = []
        for st in streams:
            r = Renderer(dev)
            r.set_stream(st.cuda_stream)
            r.upload(scene)
            rs.append(r)

        def run(k):
            for i in range(k):
                f = i % len(d_words)
                rs[i % n].update_params_device(d_words[f].data_ptr(), d_params[f].data_ptr(), d_counts[f].data_ptr(),
                                               nprim)
                rs[i % n].render_frame(cam, cfg, exact=exact, graph=True)

        run(2 * n)  # graph capture
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(streams[0])
        for st in streams[1:]:
            st.wait_event(a)
        run(frames)
        for st in streams[1:]:
            e = torch.cuda.Event()
            e.record(st)
            streams[0].wait_event(e)
        b.record(streams[0])
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / frames
        out[str(n)] = {"ms_per_frame": round(ms, 4), "Mrays_s": round(scene.width * scene.height / ms / 1e3, 1)}
        for r in rs:
            r.close()
    out["note"] = ("contexts rendering alternate frames on their own streams (device-side parameter deltas, graph "
                   "replays); throughput only -- each frame's latency stays the headline ms_per_step")
    return out


def sweep(rd_unused, exact) -> dict:
    """ms/frame vs primitive count on the other configs (device time, 10 frames)."""
    import torch

    from paper_2304_09673_b200.pipeline import RenderConfig, Renderer, Scene
    res = {}
    cfg = RenderConfig()
    stream = torch.cuda.current_stream()
    assert stream.cuda_stream != 0
    for name in ("C1", "C2", "C5", "C4"):
        s = Scene.build(name)
        r = Renderer(torch.cuda.current_device())
        r.set_stream(stream.cuda_stream)
        r.upload(s)
        for _ in range(3):
            r.render_frame(s.device_camera, cfg, exact=exact, graph=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(10):
            r.render_frame(s.device_camera, cfg, exact=exact, graph=True)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        res[name] = {"primitives": len(s.prims), "resolution": f"{s.width}x{s.height}", "ms_per_frame": round(ms, 4),
                     "Mrays_s": round(s.width * s.height / ms / 1e3, 1),
                     "stages_ms": eager_stages(r, s.device_camera, cfg, exact)}
        r.close()
        s.close()
    return res


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if os.environ.get("BT_BENCH_SHARE_GPU") == "1":
        # test mode: every rank on GPU 0, gloo -- exercises the multi-rank code
        # path (fused gather via IPC included) on a one-GPU box; not a measurement
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if os.environ.get("BT_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
