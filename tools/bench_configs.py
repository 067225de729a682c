#!/usr/bin/env python3
"""Per-config numbers for DESIGN.md: GPU join (device-resident), e2e through the
C ABI, and the CPU oracle STOMP (in full for C1-C3, a bounded row sample for
C4 and C5), for C1..C5 on one GPU.

    python tools/bench_configs.py [--configs C1,C2,C3,C4,C5] > profiles/configs_r01.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1904_12626_b200 as mp  # noqa: E402
from paper_1904_12626_b200 import datasets  # noqa: E402

sys.path.insert(0, ROOT)
from bench import cpu_sample_rate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cpu-seconds", type=float, default=6.0)
ap.add_argument("--no-cpu", action="store_true", help="GPU numbers only (quick A/B runs)")
ap.add_argument("--cpu-full", default="C1,C2,C3",
                help="configs whose CPU oracle STOMP runs in full (all rows), not sampled")
args = ap.parse_args()

for name in args.configs.split(","):
    cfg = datasets.get(name)
    a = torch.from_numpy(cfg.a).cuda()
    b = torch.from_numpy(cfg.b).cuda() if cfg.b is not None else None
    plan = mp.Plan(a, b, cfg.window, cfg.zone)
    times = []
    for r in range(args.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.prepare()
        plan.run(0, 1)
        plan.outputs()
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
    ms = min(times)
    # e2e from pinned host memory both ways (as bench.py's e2e)
    pa = torch.from_numpy(cfg.a).pin_memory().numpy()
    pb = torch.from_numpy(cfg.b).pin_memory().numpy() if cfg.b is not None else None
    La = cfg.a.size - cfg.window + 1
    names = [("mp_a", La, torch.float64), ("pi_a", La, torch.int64)]
    if cfg.b is None:
        names += [("left_a", La, torch.int64), ("right_a", La, torch.int64)]
    else:
        Lb = cfg.b.size - cfg.window + 1
        names += [("mp_b", Lb, torch.float64), ("pi_b", Lb, torch.int64)]
    host_out = {k: torch.empty(n, dtype=t, pin_memory=True).numpy() for k, n, t in names}
    tt = []
    for r in range(3):
        out = mp.join(pa, pb, cfg.window, cfg.zone, want_b=cfg.b is not None, timed=True, out=host_out)
        if r:
            tt.append(out["total_ms"])
    if args.no_cpu:
        cpu, thr, desc = None, 0, "skipped"
    elif name in args.cpu_full.split(","):
        import time as _t
        import oracle
        thr = oracle.default_threads()
        t0 = _t.perf_counter()
        oracle.stomp(cfg.a, cfg.b, cfg.window, cfg.ez, n_workers=thr)
        dt = _t.perf_counter() - t0
        cpu = cfg.cells() / dt
        desc = f"oracle STOMP (restated reference), the full join: {dt:.2f}s on {thr} threads"
    else:
        cpu, thr, desc = cpu_sample_rate(cfg, seconds_target=args.cpu_seconds)
    line = {"config": name, "workload": cfg.description, "cells": cfg.cells(),
            "gpu_ms": ms, "gpu_cells_per_s": cfg.cells() / (ms * 1e-3),
            "e2e_ms": min(tt), "e2e_cells_per_s": cfg.cells() / (min(tt) * 1e-3),
            "cpu_cells_per_s": cpu, "cpu_threads": thr, "cpu_sample": desc,
            "speedup_e2e_vs_cpu": cfg.cells() / (min(tt) * 1e-3) / cpu if cpu else None}
    print(json.dumps(line), flush=True)
    plan.close()
    del a, b
    torch.cuda.empty_cache()
