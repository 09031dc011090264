#!/usr/bin/env python
"""Instruction shares by source line of an ncu capture (executed warp
instructions, the `source` page), plus the headline counters.
    python scripts/march_lines.py gpurun_out/<rep>.ncu-rep [min_share_pct]"""
import collections
import csv
import io
import subprocess
import sys


def ncu(args):
    return list(csv.reader(io.StringIO(subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout)))


rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
raw = ncu(["-i", rep, "--page", "raw", "--csv"])
vals = dict(zip(raw[0], raw[2])) if len(raw) >= 3 else {}
for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
          "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
          "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "sass__inst_executed_local_loads",
          "smsp__thread_inst_executed_per_inst_executed.ratio"):
    print(f"{k:70s} {vals.get(k)}")
rows = ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"])
agg, txt, cur = collections.Counter(), {}, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8:
        continue
    try:
        ex, ln = int(r[7]), int(r[0])
    except ValueError:
        continue
    agg[(cur, ln)] += ex
    txt[(cur, ln)] = r[1].strip()[:90]
tot = max(1, sum(agg.values()))
byfile = collections.Counter()
for k, v in agg.items():
    byfile[k[0]] += v
print("total", tot, {k: round(100 * v / tot, 1) for k, v in byfile.most_common()})
for k, v in sorted(agg.items()):
    if 100 * v / tot >= thr:
        print(f"{k[0]:14s}{k[1]:5d} {100 * v / tot:5.1f}% {txt[k]}")
