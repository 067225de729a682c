"""Parity helpers shared by the GPU tests (test infrastructure).

Bar (BASELINE.json north_star): MP within 1e-6 relative; +inf / -1 must match
exactly; PI identical except where the two candidates' exact distances differ
by less than 1e-6 relative (checked by recomputing both by brute force).
"""
from __future__ import annotations

import numpy as np

REL = 1e-6
# Distances near 0 (exact repeats / flat windows) are compared absolutely: the
# reference's own QT formula carries ~sqrt(2m * 1e-16 * cond) there.
ABS = 1e-6


def exact_dist(x: np.ndarray, i: int, y: np.ndarray, j: int, m: int) -> float:
    """Direct z-normalised distance with the flat-window convention."""
    a = x[i:i + m]
    b = y[j:j + m]
    sa, sb = a.std(), b.std()
    fa = sa <= 1e-10 * max(1.0, abs(a.mean()))
    fb = sb <= 1e-10 * max(1.0, abs(b.mean()))
    if fa and fb:
        return 0.0
    if fa or fb:
        return float(np.sqrt(m))
    za = (a - a.mean()) / sa
    zb = (b - b.mean()) / sb
    return float(np.sqrt(min(np.sum((za - zb) ** 2), 4.0 * m)))


def close(got, ref, rel=REL, abs_=ABS):
    got = np.asarray(got)
    ref = np.asarray(ref)
    inf_ok = np.array_equal(np.isinf(got), np.isinf(ref))
    fin = np.isfinite(ref)
    err = np.abs(got[fin] - ref[fin])
    ok = err <= rel * np.abs(ref[fin]) + abs_
    return inf_ok and bool(np.all(ok)), (float(np.max(err / np.maximum(np.abs(ref[fin]), 1e-300)))
                                         if fin.any() else 0.0)


def index_mismatches(got_idx, ref_idx, rows, x, y, m, tol=REL):
    """Rows whose index differs AND whose distances are not a near-tie."""
    bad = []
    for r, gi, ri in zip(rows, got_idx, ref_idx):
        if gi == ri:
            continue
        if gi < 0 or ri < 0:
            bad.append((int(r), int(gi), int(ri)))
            continue
        dg = exact_dist(x, int(r), y, int(gi), m)
        dr = exact_dist(x, int(r), y, int(ri), m)
        if abs(dg - dr) > tol * max(dr, 1e-3) + ABS:
            bad.append((int(r), int(gi), int(ri), dg, dr))
    return bad
