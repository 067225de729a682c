#!/usr/bin/env python3
"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list.

    python tools/launch_summary.py launches.csv [--steps N]
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg, cnt = defaultdict(float), defaultdict(int)
for r in rows[start + 1:]:
    if len(r) > mv and r[mn] == "gpu__time_duration.sum":
        k = r[ki].split("(")[0]
        agg[k] += float(r[mv].replace(",", ""))
        cnt[k] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
    print(f"{k[:48]:48s} {cnt[k] // steps:4d}/step {v / 1e3 / steps:10.1f} us/step {100 * v / tot:5.1f}%")
