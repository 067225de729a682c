"""Exact anytime SCRIMP (mprof.scrimp, per-diagonal order) on C4 at 1%, 10% and 50% of the
diagonals: e2e ms per call. MPGPU_MASK_MIN_DENSITY=2 forces k_diag_join for every density."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1904_12626_b200 as mp
from paper_1904_12626_b200 import datasets
c = datasets.c4()
L = c.a.size - c.window + 1
nd = L - c.zone - 1
for frac in (100, 10, 2):
    s_size = nd // frac
    ms = []
    for r in range(4):
        t0 = time.perf_counter()
        prof = mp.scrimp(c.a, c.window, c.ez, s_size=s_size, seed=7, granularity="diagonal")
        ms.append((time.perf_counter() - t0) * 1e3)
    diags, cov = mp.scrimp_diagonals(c.a.size, c.window, c.zone, s_size, seed=7)
    cells = int(np.sum(L - diags))
    print("1/%d of diagonals: all %s e2e %.1f ms, %.3e cells/s, mp sum %.6f" % (frac, [round(v, 1) for v in ms], min(ms), cells / (min(ms) * 1e-3), float(np.sum(prof.values[np.isfinite(prof.values)]))), flush=True)
