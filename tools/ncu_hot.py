#!/usr/bin/env python3
"""Stall-sample share per code region of an ncu report (source page, SASS)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
chunk = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0x800
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc = h.index("Address"), h.index("Source")
iall, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ia], 16), r[isrc], float(r[iall] or 0), float(r[iex] or 0),
                     {h[i]: float(r[i] or 0) for i in reasons}))
    except (ValueError, IndexError):
        pass
data.sort()
base = data[0][0]
tot = sum(d[2] for d in data) or 1
reg = collections.OrderedDict()
for a, s, n, e, rs in data:
    c = reg.setdefault((a - base) // chunk, [0.0, 0.0, s.strip()[:38], collections.Counter()])
    c[0] += n
    c[1] += e
    c[3].update(rs)
for k, (n, e, s, rs) in reg.items():
    if n / tot > 0.005:
        top = ", ".join(f"{r[6:]}={v / n * 100:.0f}%" for r, v in rs.most_common(3))
        print(f"{k * chunk:#07x} {n / tot * 100:6.2f}%  inst {e:9.2e}  {s:38s} {top}")
