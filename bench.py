#!/usr/bin/env python3
"""Benchmark: matrix-profile cells/s of the B200 join (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Step = one full self-join of the workload (window stats + diagonal tiles +
finalize) with inputs resident in HBM. N=1 runs C4 (n=2^20, m=256, ECG-like,
the headline metric's shape). Under torchrun (N>1) every rank evaluates an
equal-cell shard of the diagonal work items, the packed int64 keys are
merged by RED.MIN into one key region striped over every GPU's HBM (or, with
MPGPU_SHARED_KEYS=0, min-reduced over NCCL afterwards) and rank 0 finalizes
(strong scaling: total work fixed). Rank 0 prints ONE JSON line.

`--impl reference` times the CPU restatement of the reference STOMP
(oracle/, the reference itself cannot be compiled: SURVEY.md §0) on the host
cores over a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Measured on this pool's B200 (profiles/fp64_peak_r01.jsonl, tools/microbench):
# DMUL 1.858e13/s, DFMA 1.711e13/s at 1965 MHz -> 148 SMs x 64 fp64 lanes x clock.
FP64_OPS_PER_CLK_SM = 64
N_SM = 148
FP64_PEAK_MEASURED = 1.858e13  # fp64 pipe ops/s, burst, 1965 MHz
# SURVEY.md §8(d) algorithmic cost: 6 fp64-pipe ops per cell (2 DFMA recurrence,
# 1 DMUL + 1 DFMA score, 2 compares). This build issues 4 of them on the fp64
# pipe (the two compares run as int32 high-word compares on the ALU pipe), so
# the line also carries the stricter 4-op pipe fraction.
FP64_OPS_PER_CELL_SURVEY = 6
FP64_OPS_PER_CELL_ISSUED = 4


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        mhz, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                mhz.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(mhz)}


def cpu_model() -> str:
    """Host CPU model string (the lscpu 'Model name'), for the cpu_baseline record."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_sample_rate(cfg, seconds_target=15.0, threads=None, detail=False):
    """Oracle STOMP (restated reference, oracle/) on a bounded row sample.

    Returns (unique-cells/s, threads, sample description[, detail dict with the
    rows timed, the rows of the job and the measured seconds]). Full STOMP rows cost
    L evaluations each and L rows cover the (L-z-1)(L-z)/2 unique cells, so a
    sample of R rows stands for R/L of the job. A 256-row probe sizes the
    sample to about `seconds_target` seconds."""
    import oracle
    threads = threads or oracle.default_threads()
    Lrows = (cfg.b.size - cfg.window + 1) if cfg.b is not None else cfg.a.size - cfg.window + 1
    probe = min(Lrows, 256 * threads)
    t0 = time.perf_counter()
    oracle.stomp(cfg.a, cfg.b, cfg.window, cfg.ez, n_workers=threads, row_begin=0, row_end=probe)
    dt = time.perf_counter() - t0
    rows = int(min(Lrows, max(probe, probe * seconds_target / max(dt, 1e-3))))
    if rows > probe:
        t0 = time.perf_counter()
        oracle.stomp(cfg.a, cfg.b, cfg.window, cfg.ez, n_workers=threads, row_begin=0, row_end=rows)
        dt = time.perf_counter() - t0
    else:
        rows = probe
    rate = cfg.cells() * (rows / Lrows) / dt
    desc = (f"oracle STOMP (restated reference) rows [0,{rows}) of {Lrows}, full rows, "
            f"{dt:.1f}s on {threads} threads, extrapolated to unique cells")
    if detail:
        return rate, threads, desc, {"rows_timed": rows, "rows_total": Lrows, "seconds": dt}
    return rate, threads, desc


def config_dict(cfg):
    """The `config` object of the JSON line, identical in both arms (the
    reference arm has no tile and runs on the host, but names the same workload)."""
    return {"workload": cfg.description, "config": cfg.name, "cells_per_step": cfg.cells(),
            "window": cfg.window, "exclusion_zone": cfg.zone,
            "series_checksum": checksum_of(cfg),
            "l2": "flushed between steps (256 MB write)"}


def checksum_of(cfg):
    from paper_1904_12626_b200 import datasets
    c = datasets.checksum(cfg.a)
    return c if cfg.b is None else c + "/" + datasets.checksum(cfg.b)


def flush_l2(buf):
    buf.add_(1)


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU restatement of the reference STOMP."""
    if rank != 0:
        return
    samples, secs = [], []
    threads = None
    desc = ""
    det = {}
    for s in range(args.warmup + args.steps):
        rate, threads, desc, det = cpu_sample_rate(cfg, seconds_target=args.ref_seconds, detail=True)
        if s >= args.warmup:
            samples.append(rate)
            secs.append(det["seconds"])
    v = statistics.median(samples)
    # Each step is a bounded sample of the job (the full C4 join would take
    # minutes on the host): ms_per_step is the measured wall time of that
    # sample, and `extrapolated` says how the value scales it to the job.
    line = {
        "impl": "reference", "metric": "matrix-profile cells/sec", "value": v, "unit": "cells/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(secs) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, datasets.py)",
        "config": config_dict(cfg),
        "extrapolated": {"rows_timed_per_step": det.get("rows_timed"), "rows_total": det.get("rows_total"),
                         "cells_timed_per_step": int(cfg.cells() * det.get("rows_timed", 0)
                                                     / max(1, det.get("rows_total", 1))),
                         "note": "each step times STOMP rows [0, rows_timed); value = their unique-cell "
                                 "equivalent / measured seconds (R rows of L stand for R/L of the job)"},
        "cpu_baseline": {"value": v, "unit": "cells/s", "cores": threads, "kind": "port", "sample": desc,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="cpu_baseline sample length")
    ap.add_argument("--ref-seconds", type=float, default=4.0, help="--impl reference: per-step sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)

    from paper_1904_12626_b200 import datasets
    cfg = datasets.get(args.config)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)  # rank 0 only; other ranks exit without work
        return

    import torch
    import paper_1904_12626_b200 as mp
    from paper_1904_12626_b200.distributed import (SharedKeys, merge_keys_, shared_finish,
                                                   shared_outputs, shared_prepare, sharded_prepare)
    ndev = torch.cuda.device_count()
    local = local % max(ndev, 1)  # one process per GPU; wraps only in functional tests
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("MPGPU_DIST_BACKEND", "nccl")  # gloo: functional test on 1 GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    stream = torch.cuda.Stream(dev)
    a = torch.from_numpy(cfg.a).to(dev)
    b = torch.from_numpy(cfg.b).to(dev) if cfg.b is not None else None
    with torch.cuda.stream(stream):
        plan = mp.Plan(a, b, cfg.window, cfg.zone, stream=stream)
    cells_total = plan.cells(0, 1)
    assert cells_total == cfg.cells(), (cells_total, cfg.cells())
    my_cells = plan.cells(rank, world)
    l2 = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    outs = None
    # N > 1: the keys live in one region striped over every rank's HBM (CUDA VMM,
    # 2 MB chunks round-robin) and mapped into every process; each rank's join
    # RED.MINs into it over NVLink while it computes, so the merge is fused into
    # the compute and every shard filters against the whole job's keys.
    # MPGPU_SHARED_KEYS=0 selects separate keys plus an NCCL MIN-reduce.
    shared = None
    if world > 1 and os.environ.get("MPGPU_SHARED_KEYS", "1") != "0":
        shared = SharedKeys.try_create(plan, rank, world)

    def step(ev):
        nonlocal outs
        ev[0].record(stream)
        with torch.cuda.stream(stream):
            if shared:
                shared_prepare(plan, rank, world)
            else:
                sharded_prepare(plan, rank, world)  # coarse warm start sharded + MIN-merged
        ev[1].record(stream)
        plan.run(rank, world)
        ev[2].record(stream)
        if shared:
            shared_finish(plan)
        elif world > 1:
            rk, ck = plan.keys()
            with torch.cuda.stream(stream):
                merge_keys_(rk, ck, root=0)  # NCCL ReduceOp.MIN on the packed int64 keys
        with torch.cuda.stream(stream):
            if shared:  # every rank decodes its rows into rank 0's output region
                outs = shared_outputs(plan, rank, shared=shared)
            elif rank == 0:
                outs = plan.outputs()
        ev[3].record(stream)

    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush_l2(l2)
        step(mk())
    torch.cuda.synchronize()
    # N > 1: before anything is timed, rank 0 joins the whole job alone and the
    # multi-rank profile must equal it bit for bit (the shards' cells have the
    # same arithmetic and the keys are an exact MIN). The striped-key path has
    # only ever run with several ranks on one GPU in this repo's tests, so a
    # mismatch on real peers falls back, on every rank, to separate keys plus
    # the NCCL MIN merge, and the line says so.
    check = None
    if world > 1:
        forced = [os.environ.get("MPGPU_BENCH_FORCE_MISMATCH") == "1"]  # tests: exercise the fallback

        def multi_rank_matches():
            ok = True
            if rank == 0:
                with torch.cuda.stream(stream):
                    ref_plan = mp.Plan(a, b, cfg.window, cfg.zone, stream=stream)
                    ref_plan.prepare()
                    ref_plan.run(0, 1)
                    ref = ref_plan.outputs()
                stream.synchronize()
                ok = outs is not None and all(torch.equal(outs[k], ref[k]) for k in ref)
                ref_plan.close()
            if forced[0]:
                ok, forced[0] = False, False
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                                device=dev if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            return int(flag.item()) == 1

        if cells_total > 1.5e12:
            check = "skipped (a one-rank join of this size takes too long)"
        else:
            if args.warmup == 0:
                step(mk())
                torch.cuda.synchronize()
            if multi_rank_matches():
                check = "bit-identical to rank 0's one-rank join"
            elif shared:
                shared.close()
                dist.barrier()
                shared = None
                os.environ["MPGPU_SHARED_KEYS"] = "0"  # the e2e leg follows suit
                for _ in range(max(1, args.warmup)):
                    step(mk())
                torch.cuda.synchronize()
                check = ("striped keys MISMATCHED the one-rank join; fell back to the NCCL MIN merge, "
                         + ("which matches bit for bit" if multi_rank_matches() else "which MISMATCHES too"))
            else:
                check = "MISMATCH against rank 0's one-rank join"
    launches_per_step = plan.launches() + (0 if rank else 0)

    evs = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush_l2(l2)
            e = mk()
            step(e)
            evs.append(e)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    join_ms = [e[1].elapsed_time(e[2]) for e in evs]
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms, statistics.mean(join_ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, join_avg = float(t[0]), float(t[1])
    else:
        join_avg = statistics.mean(join_ms)
    ms_per_step = total_ms / args.steps
    value = cells_total / (ms_per_step * 1e-3)

    # roofline of the dominant kernel (k_join): algorithmic fp64 pipe ops / launch time
    join_ops_per_s = my_cells * FP64_OPS_PER_CELL_SURVEY / (join_avg * 1e-3)
    issued_ops_per_s = my_cells * FP64_OPS_PER_CELL_ISSUED / (join_avg * 1e-3)
    csum = clk.summary()

    # e2e through the public host API: pinned host series -> H2D -> join -> D2H
    e2e = None
    if not args.no_e2e:
        e2e = e2e_measure(args, cfg, mp, rank, world, dev, dist)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, thr, desc = cpu_sample_rate(cfg, seconds_target=args.cpu_seconds)
        cpu = {"value": rate, "unit": "cells/s", "cores": thr, "kind": "port", "sample": desc,
               "cpu_model": cpu_model()}

    if rank == 0:
        prof = os.path.join(ROOT, "profiles", "k_join_traffic.json")
        traffic = None
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("dram_bytes_per_launch")
            except (OSError, ValueError):
                traffic = None
        line = {
            "metric": "matrix-profile cells/sec", "value": value, "unit": "cells/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, datasets.py)",
            "config": config_dict(cfg),
            "parallelism": (f"diagonal shards x{world}, " + (
                "keys striped over every GPU's HBM (CUDA VMM), RED.MIN fused into the join"
                if shared else "NCCL MIN merge")) if world > 1 else "1 GPU",
            "tile": mp.lib().mpgpu_build_info().decode(),
            "roofline": {"bound": "fp64", "kernel": "k_join", "kernel_note": "the fine join launch (plan.run), timed alone with CUDA events; the coarse warm-start join is a separate small k_join launch inside prepare, counted in value and ms_per_step",
                         "achieved": join_ops_per_s / 1e12, "peak": FP64_PEAK_MEASURED / 1e12,
                         "unit": "Tops/s (fp64 ops, SURVEY §8d: 6 per cell)",
                         "frac": join_ops_per_s / FP64_PEAK_MEASURED,
                         "frac_fp64_pipe_issued": issued_ops_per_s / FP64_PEAK_MEASURED,
                         "issued_note": "4 fp64-pipe ops/cell actually issued (2 DFMA + 2 DMUL); compares on the int pipe",
                         "cells_per_s_at_peak_6op": FP64_PEAK_MEASURED / FP64_OPS_PER_CELL_SURVEY,
                         "traffic": traffic, "join_ms_per_launch": join_avg,
                         "cells_per_launch": my_cells,
                         "peak_source": "measured fp64 microbench (profiles/fp64_peak_r01.jsonl), burst 1965 MHz"},
            "clocks": csum,
            "multi_gpu_check": check,
            "gpu_launches": launches_per_step * args.steps,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if shared:
        shared.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def e2e_measure(args, cfg, mp, rank, world, dev, dist):
    """Same metric through the host-facing API with host buffers.

    1 GPU: mpgpu_join (C ABI) from pinned host memory, outputs copied back.
    N GPUs: each rank copies the pinned series in, runs its shard, keys are
    MIN-reduced over NCCL, rank 0 finalizes and copies the profile out."""
    import torch
    L = cfg.a.size - cfg.window + 1
    pinned_a = torch.from_numpy(cfg.a).pin_memory()
    pinned_b = torch.from_numpy(cfg.b).pin_memory() if cfg.b is not None else None
    h2d = cfg.a.nbytes + (cfg.b.nbytes if cfg.b is not None else 0)
    d2h = L * 8 * (4 if cfg.b is None else 2)
    times = []
    if world == 1:
        A = pinned_a.numpy()
        B = pinned_b.numpy() if pinned_b is not None else None
        # pinned output buffers too, so both copy directions run at full speed
        names = ("mp_a", "pi_a", "left_a", "right_a") if B is None else ("mp_a", "pi_a")
        host_out = {k: torch.empty(L, dtype=torch.float64 if k == "mp_a" else torch.int64,
                                   pin_memory=True).numpy() for k in names}
        for s in range(args.warmup + args.steps):
            r = mp.join(A, B, cfg.window, cfg.zone, want_b=False, timed=True, out=host_out)
            if s >= args.warmup:
                times.append(r["total_ms"])
        t = sum(times) / len(times)
    else:
        # persistent device buffers and plan; every timed step copies the series in,
        # runs this rank's shard, MIN-reduces the keys over NCCL and (rank 0) copies
        # the profile out
        from paper_1904_12626_b200.distributed import (SharedKeys, merge_keys_, shared_finish,
                                                       shared_outputs, shared_prepare, sharded_prepare)
        stream = torch.cuda.Stream(dev)
        a = torch.empty(cfg.a.size, dtype=torch.float64, device=dev)
        b = torch.empty(cfg.b.size, dtype=torch.float64, device=dev) if pinned_b is not None else None
        with torch.cuda.stream(stream):
            plan = mp.Plan(a, b, cfg.window, cfg.zone, stream=stream)
        shared = (SharedKeys.try_create(plan, rank, world)
                  if os.environ.get("MPGPU_SHARED_KEYS", "1") != "0" else None)
        host_out = None
        for s in range(args.warmup + args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                a.copy_(pinned_a, non_blocking=True)
                if b is not None:
                    b.copy_(pinned_b, non_blocking=True)
                if shared:
                    shared_prepare(plan, rank, world)
                    plan.run(rank, world)
                    shared_finish(plan)
                else:
                    sharded_prepare(plan, rank, world)
                    plan.run(rank, world)
                    rk, ck = plan.keys()
                    merge_keys_(rk, ck, root=0)
                o = (shared_outputs(plan, rank, shared=shared) if shared
                     else plan.outputs() if rank == 0 else None)
                if rank == 0:
                    if host_out is None:
                        host_out = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in o.items()}
                    for k, v in o.items():
                        host_out[k].copy_(v, non_blocking=True)
            stream.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            tt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            if s >= args.warmup:
                times.append(float(tt[0]))
        if shared:
            shared.close()
            dist.barrier()  # every mapping closed before any rank frees its chunks
        plan.close()
        t = sum(times) / len(times)
    return {"value": cfg.cells() / (t * 1e-3), "unit": "cells/s", "ms_per_step": t,
            "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h,
            "api": "mpgpu_join (C ABI)" if world == 1 else (
                "Plan + keys striped over the GPUs (CUDA VMM)" if shared else "Plan + torch.distributed NCCL MIN")}


if __name__ == "__main__":
    main()
