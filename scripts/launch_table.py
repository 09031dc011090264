#!/usr/bin/env python
"""Per-kernel mean device time from ncu launch-list CSVs (--metrics gpu__time_duration.sum).
    python scripts/launch_table.py gpurun_out/<tag>_<cfg>_launches.csv ..."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        continue
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    t, n = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui].strip().lower()
        v = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3) * v
        k = r[ki].split("(")[0].replace("btk::", "").replace("(anonymous namespace)::", "")
        t[k] += v
        n[k] += 1
    print(f"== {path}")
    for k, v in sorted(t.items(), key=lambda kv: -kv[1] / n[kv[0]]):
        print(f"{v / n[k]:9.1f} us  x{n[k]:3d}  {k[:90]}")
