"""Parity helpers shared by the GPU tests (test infrastructure).

Bar (BASELINE.json north_star): MP within 1e-6 relative; +inf / -1 must match
exactly; PI identical except where the two candidates' exact distances differ
by less than 1e-6 relative (checked by recomputing both by brute force).
"""
from __future__ import annotations

import numpy as np

REL = 1e-6
# The only absolute slack: the fp64 rounding floor of a DIRECT z-normalised
# distance (both sides recompute near-zero distances directly). Each of the m
# z-value differences carries ~|z| * 2^-52 <= sqrt(m) * 2^-52, so an exact
# affine repeat comes out as ~m^1.5 * 2^-52 <= 1e-11 (m <= 1024) instead of 0.
# Exactly 0 (flat-vs-flat, bit-identical windows) and +inf are compared exactly.
ABS = 1e-10


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
    """MP parity: +inf and exact 0 must match exactly; finite values within
    `rel` relative (plus the direct-distance rounding floor `abs_`)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    inf_ok = np.array_equal(np.isinf(got), np.isinf(ref))
    zero_ok = np.array_equal(got == 0.0, ref == 0.0) or bool(
        np.all(np.abs(got[(got == 0.0) != (ref == 0.0)]
                      - ref[(got == 0.0) != (ref == 0.0)]) <= abs_))
    fin = np.isfinite(ref) & np.isfinite(got)
    err = np.abs(got[fin] - ref[fin])
    ok = err <= rel * np.abs(ref[fin]) + abs_
    return inf_ok and zero_ok and bool(np.all(ok)), (
        float(np.max(err / np.maximum(np.abs(ref[fin]), 1e-300))) if fin.any() else 0.0)


def index_mismatches(got_idx, ref_idx, rows, x, y, m, tol=REL):
    """Rows whose index differs AND whose exactly recomputed distances are not
    a near-tie (|d_got - d_ref| > tol * d_ref + ABS)."""
    got_idx = np.asarray(got_idx)
    ref_idx = np.asarray(ref_idx)
    rows = np.asarray(rows)
    bad = []
    for q in np.flatnonzero(got_idx != ref_idx):
        r, gi, ri = int(rows[q]), int(got_idx[q]), int(ref_idx[q])
        if gi < 0 or ri < 0:
            bad.append((r, gi, ri))
            continue
        dg = exact_dist(x, r, y, gi, m)
        dr = exact_dist(x, r, y, ri, m)
        if abs(dg - dr) > tol * dr + ABS:
            bad.append((r, gi, ri, dg, dr))
    return bad


# ---------------------------------------------------------------- multivariate
RAW_SNAP = 1e-12  # raw_distance_from_terms snap (oracle OR_RAW_SNAP)


def raw_exact(a: np.ndarray, i: int, b: np.ndarray, j: int, m: int) -> float:
    """Direct SiMPle distance: sqrt(sum_d |a_d,i - b_d,j|^2), snapped to 0
    below 1e-12 of the summed window energies. a, b: (dims, n)."""
    x = a[:, i:i + m]
    y = b[:, j:j + m]
    d2 = float(np.sum((x - y) ** 2))
    sc = float(np.sum(x * x) + np.sum(y * y))
    return 0.0 if d2 <= RAW_SNAP * sc else float(np.sqrt(d2))


def raw_index_mismatches(got_idx, ref_idx, rows, a, b, m, tol=REL):
    bad = []
    for r, gi, ri in zip(rows, got_idx, ref_idx):
        if gi == ri:
            continue
        if gi < 0 or ri < 0:
            bad.append((int(r), int(gi), int(ri)))
            continue
        dg = raw_exact(a, int(r), b, int(gi), m)
        dr = raw_exact(a, int(r), b, int(ri), m)
        if abs(dg - dr) > tol * dr + ABS:
            bad.append((int(r), int(gi), int(ri), dg, dr))
    return bad


def mstomp_order(dims, must=(), exc=()):
    must = sorted(must)  # ascending, as the oracle and the GPU order them
    order = must + [d for d in range(dims) if d not in must and d not in set(exc)]
    return order, len(must)


def mstomp_cell(x, i, j, m, order, n_must):
    """Exact selection at cell (i, j): (slot dims, prefix means) with the must
    dims first, each class ascending by distance, ties by position (stable)."""
    dist = np.array([exact_dist(x[d], i, x[d], j, m) for d in order])
    pos = list(range(len(order)))
    head = sorted(pos[:n_must], key=lambda q: (dist[q], q))
    tail = sorted(pos[n_must:], key=lambda q: (dist[q], q))
    sel = head + tail
    pk = np.cumsum(dist[sel]) / np.arange(1, len(sel) + 1)
    return [order[q] for q in sel], pk, dist[sel]


def mstomp_mismatches(got, ref, x, m, must=(), exc=(), tol=REL):
    """Compare (values, index, dim_order) triples row by row. Index and
    dim_order differences are accepted at near-ties of the exact values."""
    gv, gi, gd = got
    rv, ri, rd = ref
    order, nm = mstomp_order(x.shape[0], must, exc)
    D = len(order)
    bad = []
    ok, rel = close(gv.ravel(), rv.ravel(), tol)
    if not ok:
        bad.append(("values", rel))
    for k in range(gv.shape[0]):
        kk = min(k, D - 1)
        for c in np.flatnonzero((gi[k] != ri[k]) | (gd[k] != rd[k])):
            g, r = int(gi[k, c]), int(ri[k, c])
            if g < 0 or r < 0:
                if g != r:
                    bad.append((k, int(c), g, r))
                continue
            sg, pg, dg = mstomp_cell(x, int(c), g, m, order, nm)
            if g != r:
                _, pr, _ = mstomp_cell(x, int(c), r, m, order, nm)
                if abs(pg[kk] - pr[kk]) > tol * pr[kk] + ABS:
                    bad.append((k, int(c), g, r, pg[kk], pr[kk]))
                continue
            # same partner, different dim_order: only at a near-tie around slot kk
            if k >= D:
                bad.append((k, int(c), "dim_order", int(gd[k, c]), int(rd[k, c])))
                continue
            lo = kk - 1 if kk > 0 else kk
            hi = kk + 1 if kk + 1 < D else kk
            near = any(abs(dg[q] - dg[kk]) <= tol * dg[kk] + ABS for q in (lo, hi) if q != kk)
            if not near:
                bad.append((k, int(c), "dim_order", int(gd[k, c]), int(rd[k, c]), sg[kk]))
    return bad
