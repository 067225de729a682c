#!/usr/bin/env python3
"""Measurements for the SURVEY §8(f) rows: anytime SCRIMP, the MASS
distance-profile batch, FLUSS, mSTOMP and SiMPle. Each row is timed on the GPU (CUDA events,
inputs resident) against its roofline, next to the CPU oracle on a bounded
sample.

    python tools/bench_next.py > profiles/next_r01.jsonl
"""
import json
import os
import sys
import time
import ctypes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (checker / CPU baseline only)
import paper_1904_12626_b200 as mp  # noqa: E402
from paper_1904_12626_b200 import datasets  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
HBM_GBS = PEAKS.get("hbm_gbs", 6553.0)
DFMA_PER_S = 1.711e13  # measured DFMA rate, profiles/fp64_peak_r01.jsonl (1965 MHz)
THREADS = oracle.default_threads()


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def emit(d):
    print(json.dumps(d), flush=True)


def anytime_scrimp():
    """Anytime SCRIMP on C4 at 10% of the diagonals, both granularities: the band
    fast path (the same k_join over a seeded band subset) and the reference's
    exact per-diagonal order (k_diag_join, one diagonal per lane)."""
    c = datasets.c4()
    L = c.a.size - c.window + 1
    nd = L - c.zone - 1
    s_size = nd // 10
    bands, coverage = mp.scrimp_bands(c.a.size, c.window, c.zone, s_size, seed=7)
    diags_exact, cov_exact = mp.scrimp_diagonals(c.a.size, c.window, c.zone, s_size, seed=7)
    # CPU: the oracle's SCRIMP loop over a few of the band diagonals
    diags = np.arange(c.zone + 1 + 256 * int(bands[0]), c.zone + 1 + 256 * int(bands[0]) + 64)
    t0 = time.perf_counter()
    oracle.scrimp_diagonals(c.a, c.window, diags, threads=THREADS)
    cpu_s = time.perf_counter() - t0
    cpu_cells = sum(L - int(k) for k in diags)
    for gran in ("band", "diagonal"):
        ms = []
        for r in range(3):
            t0 = time.perf_counter()
            prof = mp.scrimp(c.a, c.window, c.ez, s_size=s_size, seed=7, granularity=gran)
            ms.append((time.perf_counter() - t0) * 1e3)
        if gran == "band":  # cells evaluated: the chosen bands' diagonals, (L - k) each
            cells = 0
            for b in bands:
                k0 = c.zone + 1 + 256 * int(b)
                cells += sum(L - k for k in range(k0, min(k0 + 256, L)))
        else:
            cells = int(np.sum(L - diags_exact))
        e2e = float(np.median(ms))
        emit({"row": "8f.1 anytime SCRIMP", "granularity": gran,
              "workload": "C4, s_size = 10% of diagonals, seed 7",
              "coverage": prof.coverage, "bands": int(bands.size) if gran == "band" else None,
              "diagonals": int(diags_exact.size) if gran == "diagonal" else None, "cells": cells,
              "e2e_ms": e2e, "e2e_cells_per_s": cells / (e2e * 1e-3),
              "note": "e2e through mprof.scrimp (host buffers, includes stats, warm start, finalize)",
              "cpu_cells_per_s": cpu_cells / cpu_s, "cpu_threads": THREADS,
              "cpu_sample": f"oracle SCRIMP loop over {diags.size} diagonals"})


def mass_batch():
    """MASS distance-profile batch: Q = 64 queries from the C4 series against every window."""
    c = datasets.c4()
    m = c.window
    x = torch.from_numpy(c.a).cuda()
    L = c.a.size - m + 1
    Q = 64
    pos = torch.from_numpy(np.random.default_rng(3).choice(L, Q, replace=False).astype(np.int64)).cuda()
    out = torch.empty((Q, L), dtype=torch.float64, device="cuda")  # allocated outside the timing

    def run():
        mp.distance_profiles(x, m, positions=pos, zone=c.zone, out=out)

    ms = ev_time(run)
    dfma = Q * L * m
    # CPU: oracle direct distance profile of 2 queries on all threads
    t0 = time.perf_counter()
    for q in pos[:2].cpu().numpy():
        oracle.mass_distance_profile(c.a[q:q + m], c.a, query_index=int(q), zone=c.zone, threads=THREADS)
    cpu_s = (time.perf_counter() - t0) / 2
    emit({"row": "8f.2 MASS distance-profile batch", "workload": f"C4 series, Q={Q} queries, m={m}, L={L}",
          "gpu_ms": ms, "outputs_per_s": Q * L / (ms * 1e-3),
          "roofline": {"bound": "fp64", "achieved": dfma / (ms * 1e-3) / 1e12, "peak": DFMA_PER_S / 1e12,
                       "unit": "T DFMA/s (m per output)", "frac": dfma / (ms * 1e-3) / DFMA_PER_S},
          "cpu_outputs_per_s": L / cpu_s, "cpu_threads": THREADS,
          "cpu_sample": "oracle mass_distance_profile, 2 queries"})


def fluss_row():
    """FLUSS arc count + CAC over a PI of L = 2^23 windows (HBM / latency bound)."""
    L = 1 << 23
    window = 128
    g = np.random.default_rng(5)
    pi = g.integers(0, L, L).astype(np.int64)
    ix = torch.from_numpy(pi).cuda()
    arcs = torch.empty(L, dtype=torch.int64, device="cuda")
    cac = torch.empty(L, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()

    def run():
        rc = mp.lib().mpgpu_fluss(mp._dev_ptr(ix), L, window, mp._dev_ptr(arcs), mp._dev_ptr(cac), 0,
                                  ctypes.c_void_p(st.cuda_stream))
        assert rc == 0

    ms = ev_time(run)
    alg_bytes = L * (8 + 8 + 8)  # read PI, write arc counts, write CAC
    t0 = time.perf_counter()
    a = oracle.fluss_arc_count(pi)
    oracle.fluss_cac(a, window)
    cpu_s = time.perf_counter() - t0
    emit({"row": "8f.4 FLUSS arc count + CAC", "workload": f"random PI, L={L}, window={window}",
          "gpu_ms": ms, "windows_per_s": L / (ms * 1e-3),
          "roofline": {"bound": "hbm", "achieved": alg_bytes / (ms * 1e-3) / 1e9, "peak": HBM_GBS,
                       "unit": "GB/s (24 algorithmic B per window)",
                       "frac": alg_bytes / (ms * 1e-3) / 1e9 / HBM_GBS},
          "cpu_windows_per_s": L / cpu_s, "cpu_threads": 1, "cpu_sample": "oracle numpy restatement, full L"})


def _unique_cells(L, zone):
    r = L - zone - 1
    return r * (r + 1) // 2 if r > 0 else 0


def multivariate_row(kind, d, n, m, ops_per_cell, ops_note):
    """mSTOMP / SiMPle self-join on d seeded random walks (no BASELINE config
    names these; SPEC.md:225-243 shapes). GPU: device time of the call's
    kernels (stats + diagonal kernel + finalize, CUDA events inside the
    library) and wall time through the API from host buffers. CPU: the
    oracle's STOMP-order loop over a bounded row sample on all host threads."""
    g = np.random.default_rng(2018 + d)
    x = np.cumsum(g.standard_normal((d, n)), axis=1)
    L = n - m + 1
    zone = mp.zone_size(m, 0.5)
    f = (lambda: mp.mstomp(x, m, 0.5, timed=True)) if kind == "mstomp" else \
        (lambda: mp.simple_join(x, None, m, 0.5, timed=True))
    f()
    ks, ws = [], []
    for _ in range(5):
        t0 = time.perf_counter()
        r = f()
        ws.append(time.perf_counter() - t0)
        ks.append(r.kernel_ms)
    k_ms, w_s = float(np.median(ks)), float(np.median(ws))
    cells = _unique_cells(L, zone)
    rows = max(THREADS, min(L, int(2e9 / (L * d * (12 if kind == "mstomp" else 4)))))
    t0 = time.perf_counter()
    if kind == "mstomp":
        oracle.mstomp(x, m, 0.5, n_workers=THREADS, row_begin=0, row_end=rows)
    else:
        oracle.simple_join(x, None, m, 0.5, n_workers=THREADS, row_begin=0, row_end=rows)
    cpu_s = time.perf_counter() - t0
    ach = cells * ops_per_cell / (k_ms * 1e-3)
    emit({"row": f"8f.4 {'mSTOMP' if kind == 'mstomp' else 'SiMPle'} (d={d})",
          "workload": f"self-join, {d} random walks, n={n}, m={m}, zone={zone}",
          "cells": cells, "gpu_ms": k_ms, "cells_per_s": cells / (k_ms * 1e-3),
          "e2e_ms": 1e3 * w_s, "e2e_cells_per_s": cells / w_s,
          "roofline": {"bound": "fp64", "achieved": ach / 1e12, "peak": 18.58,
                       "unit": f"Tops/s ({ops_per_cell} fp64 ops per cell: {ops_note})",
                       "frac": ach / 18.58e12},
          "cpu_cells_per_s": cells * rows / L / cpu_s, "cpu_threads": THREADS,
          "cpu_sample": f"oracle {kind} rows [0,{rows}) of {L}, full rows, unique-cell equivalent"})


if __name__ == "__main__":
    oracle.build()
    mp.lib()
    only = sys.argv[1:]
    if not only or "scrimp" in only:
        anytime_scrimp()
    if not only or "mass" in only:
        mass_batch()
    if not only or "fluss" in only:
        fluss_row()
    if not only or "multi" in only:
        # one admissible dim runs on k_join: SURVEY §8(d)'s 6 fp64-pipe ops per cell
        multivariate_row("mstomp", 1, 1 << 16, 256, 6, "k_join (one admissible dim): SURVEY 8(d) count")
        multivariate_row("mstomp", 3, 1 << 16, 256, 36,
                         "per dim 2 recurrence + 2 normalise + 1 distance + 5 sqrt + 2 prefix mean")
        multivariate_row("mstomp", 8, 1 << 15, 128, 96,
                         "per dim 2 recurrence + 2 normalise + 1 distance + 5 sqrt + 2 prefix mean")
        for d, n, m in ((1, 1 << 17, 256), (3, 1 << 16, 256), (8, 1 << 16, 128), (12, 1 << 15, 64)):
            multivariate_row("simple", d, n, m, 2 * d + 2, "2 per dim recurrence + add + distance")
