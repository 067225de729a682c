#!/usr/bin/env python3
"""Per-instruction warp-state (pc sampling) attribution of an ncu --set full
report with --import-source on: stall-reason shares per code region and per
opcode in a given address range (e.g. k_join's fast block).

    python tools/ncu_opcode_stalls.py profiles/prof_kjoin_r02.ncu-rep [lo_hex hi_hex]
"""
import collections
import csv
import io
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi]
    ia, isrc = h.index("Address"), h.index("Source")
    iall = h.index("Warp Stall Sampling (All Samples)")
    iex = h.index("Instructions Executed")
    reasons = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    data = []
    for r in rows[hi + 1:]:
        try:
            data.append((int(r[ia], 16), r[isrc].strip(), float(r[iall] or 0), float(r[iex] or 0),
                         {h[i][6:]: float(r[i] or 0) for i in reasons}))
        except (ValueError, IndexError):
            pass
    data.sort()
    return data


def opcode(src):
    t = src.split()
    t = t[1:] if t and t[0].startswith("@") else t
    return t[0].split(".")[0] if t else "?"


def main():
    rep = sys.argv[1]
    data = load(rep)
    base = data[0][0]
    tot = sum(d[2] for d in data) or 1.0
    lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else None
    hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else None
    if lo is None:  # the densest DFMA/DMUL window of 0x1800 bytes
        fp = [(d[0] - base, d[2]) for d in data if opcode(d[1]) in ("DFMA", "DMUL")]
        best, lo = 0.0, 0
        for a, _ in fp:
            s = sum(w for b, w in fp if a <= b < a + 0x1800)
            if s > best:
                best, lo = s, a
        hi = lo + 0x1800
    sel = [d for d in data if lo <= d[0] - base < hi]
    share = sum(d[2] for d in sel) / tot
    print(f"report {rep}: {len(data)} instructions, {tot:.0f} samples")
    print(f"region [{lo:#x}, {hi:#x}): {len(sel)} instructions, {share * 100:.1f}% of all samples")
    agg = collections.Counter()
    for d in sel:
        agg.update(d[4])
    s = sum(agg.values()) or 1.0
    print("stall reasons in the region: " + ", ".join(f"{k} {v / s * 100:.1f}%" for k, v in agg.most_common(9)))
    op = collections.defaultdict(lambda: [0.0, 0, collections.Counter()])
    for d in sel:
        o = op[opcode(d[1])]
        o[0] += d[2]
        o[1] += 1
        o[2].update(d[4])
    print(f"{'opcode':10s} {'count':>5s} {'samples%':>9s}  top stalls")
    for k, (n, c, rs) in sorted(op.items(), key=lambda kv: -kv[1][0]):
        if n / tot < 0.002:
            continue
        top = ", ".join(f"{r} {v / n * 100:.0f}%" for r, v in rs.most_common(3))
        print(f"{k:10s} {c:5d} {n / tot * 100:9.2f}  {top}")


if __name__ == "__main__":
    main()
