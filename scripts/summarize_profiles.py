#!/usr/bin/env python
"""Summarise a GPU round's ncu artefacts (gpurun_out/<tag>_*) into profiles/.

    python scripts/summarize_profiles.py <tag> <round-prefix>   e.g.  g11 r01

Writes profiles/<round>_<tag>_launches.md (per-kernel device time from the
`--metrics gpu__time_duration.sum` launch list: cold-cache, serialised -- use
the SHARES) and profiles/<round>_<tag>_<kernel>.md (key metrics, stall reasons
and hottest source lines of each `--set full` capture), plus the bench line.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp instruction"),
    ("sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread FFMA"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread FFMA (smsp)"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread FADD (smsp)"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread FMUL (smsp)"),
    ("sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread FADD"),
    ("sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread FMUL"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("sass__inst_executed_local_loads", "local loads (warp)"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    if len(rows) < 3:
        return {}, {}
    names, units, vals = rows[0], rows[1], rows[2]
    return dict(zip(names, vals)), dict(zip(names, units))


def hot_lines(rep, n=20):
    rows = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"])
    agg, samp, txt, cur = collections.Counter(), collections.Counter(), {}, None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] in ("Line No", "Function Name", ""):
            continue
        try:
            ex, sm = int(r[7]), int(r[4])
        except ValueError:
            continue
        k = (cur, int(r[0]))
        agg[k] += ex
        samp[k] += sm
        txt[k] = r[1].strip()[:90]
    tot, ts = max(1, sum(agg.values())), max(1, sum(samp.values()))
    return [(v / ts * 100, agg[k] / tot * 100, k, txt[k]) for k, v in samp.most_common(n)]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        name = name.replace("btk::<unnamed>::", "").replace("<unnamed>::", "").replace("btk::", "")
        agg[name][0] += 1
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale
    return agg


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# {rnd} / {tag}: per-kernel device time (ncu launch list)", ""]
    bench = os.path.join(OUT, f"{tag}_bench.txt")
    if os.path.exists(bench):
        for l in open(bench):
            if l.startswith("{"):
                d = json.loads(l)
                lines += [f"bench: {d['value']} {d['unit']}, {d['ms_per_step']} ms/frame, stages {d.get('stages_ms')}",
                          f"roofline: {json.dumps(d.get('roofline'))}", f"frame_stats: {d.get('frame_stats')}", ""]
    lp = os.path.join(OUT, f"{tag}_launches.csv")
    if os.path.exists(lp):
        agg = launches(lp)
        # the bench's own measurement helpers (FP32 peak microbenchmark, L2
        # flush) run in the same process but are not part of a frame
        helper = lambda k: "k_ffma_peak" in k or "FillFunctor" in k  # noqa: E731
        total = sum(v[1] for k, v in agg.items() if not helper(k))
        lines += ["Cold-cache, serialised per-launch times (`ncu --metrics gpu__time_duration.sum --clock-control none`);",
                  "compare shares, not absolutes. Shares are of the frame kernels only.", "",
                  "| kernel | launches | us/launch | share |", "|---|---|---|---|"]
        for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            share = "(bench helper, not in the frame)" if helper(k) else f"{us / total * 100:.1f}%"
            lines.append(f"| `{k}` | {n} | {us / n:.1f} | {share} |")
    open(os.path.join(PROF, f"{rnd}_{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    traffic = {}
    for rep in sorted(f for f in os.listdir(OUT) if f.startswith(tag + "_prof_") and f.endswith(".ncu-rep")):
        kern = rep[len(tag) + 6:-8]
        m, u = raw_metrics(os.path.join(OUT, rep))
        out = [f"# {rnd} / {tag}: ncu --set full capture of {kern}", "", "| metric | value | unit |", "|---|---|---|"]
        for key, label in KEYS:
            if key in m:
                out.append(f"| {label} (`{key}`) | {m[key]} | {u.get(key, '')} |")
        stalls = sorted(((float(v), k) for k, v in m.items() if k.startswith("smsp__average_warps_issue_stalled_")
                         and "not_issued" not in k and v.replace(".", "").isdigit()), reverse=True)[:8]
        out += ["", "Top stall reasons (warps per issue slot):", ""]
        out += [f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.2f}"
                for v, k in stalls]
        out += ["", "Hottest source lines (share of stall samples, share of executed instructions):", ""]
        for s_, e_, k, t in hot_lines(os.path.join(OUT, rep)):
            out.append(f"- {s_:5.1f}% samples, {e_:5.1f}% inst — {k[0]}:{k[1]} `{t}`")
        open(os.path.join(PROF, f"{rnd}_{tag}_{kern}.md"), "w").write("\n".join(out) + "\n")
        try:
            rd_, wr_ = float(m["dram__bytes_read.sum"]), float(m["dram__bytes_write.sum"])
            mul = lambda k: {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(k, "byte"), 1)  # noqa: E731
            traffic[kern] = {"dram_bytes_per_launch": rd_ * mul("dram__bytes_read.sum") + wr_ * mul("dram__bytes_write.sum"),
                             "duration_us": float(m.get("gpu__time_duration.sum", "nan")),
                             "source": f"profiles/{rnd}_{tag}_{kern}.md (ncu --set full)"}
            fk = "smsp__sass_thread_inst_executed_op_%s_pred_on.sum"
            if fk % "ffma" in m:  # executed FP32 flops per launch: 2 FFMA + FADD + FMUL (SURVEY 8(d) cross-check)
                traffic[kern]["fp32_executed_flops"] = (2 * float(m[fk % "ffma"]) + float(m[fk % "fadd"]) +
                                                        float(m[fk % "fmul"]))
        except (KeyError, ValueError):
            pass
    if traffic:
        import json as _json
        path = os.path.join(PROF, "latest_traffic.json")
        merged = _json.load(open(path)) if os.path.exists(path) else {}
        # per (kernel, config tag) -- the bench reads the capture of its own
        # config ("k_march@c3") -- and under the bare kernel name (latest)
        merged.update(traffic)
        merged.update({f"{k}@{tag}": v for k, v in traffic.items()})
        open(path, "w").write(_json.dumps(merged, indent=1) + "\n")
    print("written to", PROF)


if __name__ == "__main__":
    main()
