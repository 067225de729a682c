#!/usr/bin/env python3
"""Generate the golden fixtures that pin the CPU oracle (test infrastructure).

Two kinds of fixture, both committed next to this script:

* ``spec_kat.json`` — the known-answer examples the reference specifies for
  this path, transcribed from /root/reference/SPEC.md (line numbers cited per
  entry). The reference ships no executable tests or golden files (SURVEY.md
  §4), so these prose examples are its only pinned answers.
* ``brute_*.npz`` — seeded small inputs with matrix profiles computed by an
  independent numpy brute force (direct per-window z-normalisation, the
  reference oracle's definition), written without any code
  from oracle/ or the product. Flat-window convention per SPEC.md "DESIGN
  DECISIONS"; ties resolve to the smallest index.

Run: python tests/golden/make_golden.py  (deterministic; rewrites the files)
"""
from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
FLAT_REL = 1e-10


def znorm_windows(x: np.ndarray, w: int):
    win = np.lib.stride_tricks.sliding_window_view(x, w)
    mu = win.mean(axis=1)
    sd = np.sqrt(((win - mu[:, None]) ** 2).mean(axis=1))
    flat = sd <= FLAT_REL * np.maximum(1.0, np.abs(mu))
    z = np.zeros_like(win)
    nz = ~flat
    z[nz] = (win[nz] - mu[nz, None]) / sd[nz, None]
    return z, flat


def brute(a: np.ndarray, b: np.ndarray | None, w: int, ez: float):
    """Matrix profile of a (against b, or itself) by direct distances."""
    self_join = b is None
    za, fa = znorm_windows(a, w)
    zb, fb = (za, fa) if self_join else znorm_windows(b, w)
    zone = int(np.floor(w * ez + 0.5)) if self_join else 0
    La, Lb = za.shape[0], zb.shape[0]
    # squared distances via the identity |za-zb|^2 = 2w - 2 za.zb for unit windows
    d2 = 2.0 * w - 2.0 * (za @ zb.T)
    d2 = np.clip(d2, 0.0, 4.0 * w)
    d = np.sqrt(d2)
    # flat-window convention
    both = fa[:, None] & fb[None, :]
    one = fa[:, None] ^ fb[None, :]
    d[both] = 0.0
    d[one] = np.sqrt(w)
    # exact direct recomputation near the minimum is not needed at these sizes:
    # recompute every entry directly for full fidelity
    for i in range(La):
        if fa[i]:
            continue
        diff = za[i][None, :] - zb
        dd = np.sqrt(np.minimum(np.sum(diff * diff, axis=1), 4.0 * w))
        keep = ~fb
        d[i, keep] = dd[keep]
    if self_join:
        idx = np.arange(La)
        excl = np.abs(idx[:, None] - idx[None, :]) <= zone
        d[excl] = np.inf
    mp = d.min(axis=1)
    pi = np.where(np.isfinite(mp), d.argmin(axis=1), -1)
    out = {"mp": mp, "pi": pi.astype(np.int64)}
    if self_join:
        left = np.where(np.tril(np.ones((La, La), bool), -1), d, np.inf)
        right = np.where(np.triu(np.ones((La, La), bool), 1), d, np.inf)
        lmin, rmin = left.min(axis=1), right.min(axis=1)
        out["left"] = np.where(np.isfinite(lmin), left.argmin(axis=1), -1).astype(np.int64)
        out["right"] = np.where(np.isfinite(rmin), right.argmin(axis=1), -1).astype(np.int64)
    return out


def spec_kat():
    return {
        "source": "/root/reference/SPEC.md (prose examples; no executable reference tests exist)",
        "rolling_mean_std": [
            {"ts": [1, 1, 1, 1, 1], "w": 4, "means": [1, 1], "stds": [0, 0], "ref": "SPEC.md:76"},
            {"ts": [0, 1, 0, 1, 0, 1], "w": 4, "means": [0.5, 0.5, 0.5], "stds": [0.5, 0.5, 0.5],
             "ref": "SPEC.md:77"},
        ],
        "sliding_dot_product": [
            {"query": [1, 0], "ts": [3, 4, 5], "out": [3, 4], "ref": "SPEC.md:86"},
        ],
        "zone_size": [
            {"w": 50, "fraction": 0.5, "zone": 25, "ref": "SPEC.md:116"},
            {"w": 80, "fraction": 0.5, "zone": 40, "ref": "SPEC.md:117"},
            {"w": 50, "fraction": 0.25, "zone": 13, "ref": "SPEC.md:118"},
        ],
        "exclusion_zone": [
            {"length": 9922, "center": 584, "zone": 40, "finite_remaining": 9841,
             "inf_range": [544, 624], "ref": "SPEC.md:128"},
        ],
        "profile_size": [
            {"n": 10001, "w": 80, "ez": 0.5, "size": 9922, "zone": 40, "ref": "SPEC.md:202"},
            {"n": 904, "w": 50, "ez": 0.25, "size": 855, "zone": 13, "ref": "SPEC.md:212"},
        ],
        "stomp_constant": {"n": 64, "w": 8, "ez": 0.5, "value": 0.0, "ref": "SPEC.md:213"},
        "ab_self_identity": {"ref": "SPEC.md:192", "value": 0.0, "index": "i"},
    }


def main():
    with open(os.path.join(HERE, "spec_kat.json"), "w") as f:
        json.dump(spec_kat(), f, indent=1)
    g = np.random.Generator(np.random.MT19937(1904))
    cases = []
    # self-joins: random walks of assorted sizes / windows / zones
    for k, (n, w, ez) in enumerate([(300, 20, 0.5), (512, 32, 0.25), (700, 50, 0.0), (400, 8, 0.5)]):
        a = np.cumsum(g.standard_normal(n))
        cases.append((f"brute_self_{k}", a, None, w, ez))
    # flat runs + planted repeat
    a = np.cumsum(g.standard_normal(600))
    a[100:180] = a[100]
    a[400:430] = -3.0
    a[250:290] = a[480:520] + 2.5  # affine copy: distance 0 after z-normalisation
    cases.append(("brute_self_flat_planted", a, None, 24, 0.5))
    # AB-join
    a = np.cumsum(g.standard_normal(400))
    b = np.cumsum(g.standard_normal(250))
    cases.append(("brute_ab_0", a, b, 30, 0.0))
    for name, a, b, w, ez in cases:
        out = brute(a, b, w, ez)
        arrs = {"a": a, "w": np.int64(w), "ez": np.float64(ez), **out}
        if b is not None:
            arrs["b"] = b
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrs)
        print(name, a.size, None if b is None else b.size, w, ez)


if __name__ == "__main__":
    main()
