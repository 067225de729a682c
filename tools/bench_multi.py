"""Timing of the multivariate joins (SiMPle, mSTOMP) on one GPU through the
C ABI: device time (kernel_ms: statistics + diagonal kernel + finalize) and
call wall time, cells/s in unique-pair cells. Prints JSON lines."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1904_12626_b200 as mp


def cells_self(L, zone):
    r = L - zone - 1
    return r * (r + 1) // 2 if r > 0 else 0


def run(kind, d, n, w, reps=3):
    g = np.random.default_rng(2018)
    x = np.cumsum(g.standard_normal((d, n)), axis=1)
    L = n - w + 1
    zone = mp.zone_size(w, 0.5)
    f = (lambda: mp.simple_join(x, None, w, 0.5, timed=True)) if kind == "simple" else \
        (lambda: mp.mstomp(x, w, 0.5, timed=True))
    f()
    ks, ws = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = f()
        ws.append(time.perf_counter() - t0)
        ks.append(r.kernel_ms)
    cells = cells_self(L, zone)
    k = float(np.median(ks))
    return {"kind": kind, "dims": d, "n": n, "window": w, "cells": cells, "kernel_ms": k,
            "cells_per_s": cells / (k * 1e-3), "wall_ms": 1e3 * float(np.median(ws)),
            "e2e_cells_per_s": cells / float(np.median(ws))}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--case", action="append", default=[],
                    help="kind,dims,n,window (repeatable); replaces the default list")
    a = ap.parse_args()
    cases = [("simple", 3, 1 << 16, 256), ("mstomp", 3, 1 << 16, 256)]
    if a.case:
        cases = [(c.split(",")[0], *map(int, c.split(",")[1:])) for c in a.case]
    elif not a.quick:
        cases += [("simple", 1, 1 << 17, 256), ("simple", 12, 1 << 15, 64),
                  ("mstomp", 1, 1 << 17, 256), ("mstomp", 8, 1 << 15, 128)]
    for c in cases:
        print(json.dumps(run(*c)), flush=True)
