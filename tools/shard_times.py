#!/usr/bin/env python3
"""Per-shard timing of the N-GPU join, measured on ONE GPU.

Every rank of an N-GPU run executes the same kernels on its own device: the
sharded prepare (its 1/N of the coarse warm-start join, then the warm-start
finish), its shard of the diagonal work items, and rank 0 the finalize. Their
only exchange is the MIN of the packed keys (coarse keys inside prepare, full
keys after the join). This script runs each shard of each N in turn on one
GPU, with the keys reset to their post-warm-start state before every shard
(so a shard never benefits from another's results), and times each phase
with CUDA events:

    step_N = max_s coarse_s + finish + max_s join_s + merge_est + finalize

merge_est is the key MIN over NVLink estimated from bytes (16 B per window,
at 450 GB/s, half the NVLink 5 per-direction rate); it is the one unmeasured
term. efficiency_N = step_1 / (N * step_N), the figure the driver computes
from bench.py lines at N GPUs.

    python tools/shard_times.py [--config C4] [--ns 1,2,4,8] > profiles/shard_times_r01.jsonl

--traffic prints the peer-read model of the striped key region instead: the
chunk owners mpgpu_plan_key_region_owners picks for each N, the busiest GPU's
share of all key reads, and from the measured one-GPU join rate the remote
key bytes per cell of a rank and the peer-read bandwidth the busiest GPU
serves (against the single-owner layout, where one GPU serves them all).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1904_12626_b200 as mp  # noqa: E402
from paper_1904_12626_b200 import datasets  # noqa: E402

NVLINK_MERGE_GBS = 450.0
# k_join's per-tile prefetch: 32 row keys + 32 column keys (8 B each) per
# 32 row-steps x 256 diagonals = 8192 cells
KEY_BYTES_PER_CELL = 64 * 8 / 8192.0


def traffic(plan, cfg, stream, ns):
    import paper_1904_12626_b200 as mp
    gran = int(mp.lib().mpgpu_stripes_granularity(plan.device))
    plan.prepare()
    torch.cuda.synchronize()
    join_ms = timed(stream, lambda: plan.run(0, 1))
    rate = cfg.cells() / (join_ms * 1e-3)  # cells/s of one GPU
    read_gbs = rate * KEY_BYTES_PER_CELL / 1e9
    for N in ns:
        owners, share = plan.key_region_owners(gran, N)
        counts = [owners.count(r) for r in range(N)]
        print(json.dumps({
            "config": cfg.name, "n_ranks": N, "region_bytes": plan.key_region_bytes(),
            "chunk_bytes": gran, "chunks": len(owners), "chunks_per_rank": counts,
            "busiest_rank_share_of_key_reads": share,
            "key_bytes_per_cell": KEY_BYTES_PER_CELL,
            "remote_key_bytes_per_cell_per_rank": KEY_BYTES_PER_CELL * (N - 1) / N,
            "one_gpu_cells_per_s": rate, "key_read_gbs_per_rank": read_gbs,
            "busiest_gpu_peer_reads_gbs": read_gbs * (N - 1) * share,
            "single_owner_peer_reads_gbs": read_gbs * (N - 1),
            "note": "striped: every other rank sends `share` of its key reads to the busiest GPU; "
                    "single owner (round 1): all of them to rank 0"}), flush=True)


def timed(stream, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--ns", default="1,2,4,8")
    ap.add_argument("--shared", action="store_true",
                    help="shared-key phases: prepare_shared / seed_shared per shard, then the shard "
                         "joins run one after another into the same keys (no reset between them)")
    ap.add_argument("--traffic", action="store_true", help="peer-read model of the striped key region")
    args = ap.parse_args()
    cfg = datasets.get(args.config)
    stream = torch.cuda.Stream()
    a = torch.from_numpy(cfg.a).cuda()
    b = torch.from_numpy(cfg.b).cuda() if cfg.b is not None else None
    with torch.cuda.stream(stream):
        plan = mp.Plan(a, b, cfg.window, cfg.zone, stream=stream)
    # warm-up: one full single-rank step
    plan.prepare(); plan.run(0, 1); plan.outputs(); torch.cuda.synchronize()
    if args.traffic:
        traffic(plan, cfg, stream, [int(v) for v in args.ns.split(",")])
        plan.close()
        return
    key_bytes = (plan.La + plan.Lb) * 8
    merge_est = key_bytes / (NVLINK_MERGE_GBS * 1e9) * 1e3
    step1 = None
    if args.shared:
        plan.coarse_key_ptrs()  # coarse keys shared too: prepare_shared stops before the coarse join
        for N in [int(v) for v in args.ns.split(",")]:
            plan.reset_keys()
            prep = [timed(stream, lambda: plan.prepare_shared(s, N)) for s in range(N)]
            # the coarse shards, one after another into the one coarse key set (the
            # first sees only its own coarse cells, later ones the others' as well)
            plan.prepare_shared(0, N)
            coarse = [timed(stream, lambda: plan.coarse_run(s, N)) for s in range(N)]
            seed = []
            for s in range(N):  # each shard's seeding, from complete coarse keys
                plan.prepare_shared(0, N)
                plan.coarse_run(0, 1)
                seed.append(timed(stream, lambda: plan.seed_shared(s, N)))
            # the joins start from the whole job's warm start (every shard's seeds)
            plan.reset_keys()
            plan.prepare_shared(0, 1)
            plan.coarse_run(0, 1)
            plan.seed_shared(0, 1)
            torch.cuda.synchronize()
            joins = [timed(stream, lambda: plan.run(s, N)) for s in range(N)]
            outs = plan.outputs()
            fin = timed(stream, plan.outputs)
            names = ("mp_a", "pi_a", "left_a", "right_a") if plan.self_join else ("mp_a", "pi_a")
            fin_sh = [timed(stream, lambda: plan.finalize_shard(
                s, N, *[outs[k] for k in names[:2]],
                *([outs[k] for k in names[2:]] if plan.self_join else [None, None]),
                *([None, None] if plan.self_join else [outs["mp_b"], outs["pi_b"]]))) for s in range(N)]
            # a concurrent run: every shard starts against the warm start, but all
            # shards' records land in the one key set as they go, so the job's
            # key state at any moment matches a one-GPU run at the same fraction
            # of the work (items are dealt round-robin in cost order). The later
            # shards of the sequence (which see the earlier shards' final keys)
            # bound the join from below, the first (warm start only) from above.
            later = joins[1:] if N > 1 else joins
            barrier_ms = 0.03  # per host barrier (gloo/NCCL over loopback, measured ~20-40 us)
            step_lo = max(prep) + max(coarse) + max(seed) + max(later) + max(fin_sh) + 4 * barrier_ms
            step_hi = max(prep) + max(coarse) + max(seed) + joins[0] + max(fin_sh) + 4 * barrier_ms
            print(json.dumps({"config": cfg.name, "mode": "shared keys, shards in sequence", "n_shards": N,
                              "prepare_shared_ms": prep, "coarse_run_ms": coarse,
                              "seed_shared_ms": seed, "join_ms": joins,
                              "finalize_ms": fin, "finalize_shard_ms": fin_sh,
                              "step_pred_ms_range": [step_lo, step_hi],
                              "note": "step = prepare + coarse shard + seeding + join shard + finalize shard "
                                      "+ 4 barriers; low end: join as the later shards (keys as a concurrent "
                                      "run sees them), high end: the first shard (warm start only)"}),
                  flush=True)
        plan.close()
        return
    for N in [int(v) for v in args.ns.split(",")]:
        coarse, joins = [], []
        for s in range(N):
            coarse.append(timed(stream, lambda: plan.prepare_shard(s, N)))
        finish = timed(stream, plan.prepare_finish)  # coarse keys of all shards are merged in place
        for s in range(N):
            plan.prepare()  # reset the keys to the post-warm-start state
            torch.cuda.synchronize()
            joins.append(timed(stream, lambda: plan.run(s, N)))
        fin = timed(stream, plan.outputs)
        step = max(coarse) + finish + max(joins) + (merge_est if N > 1 else 0.0) + fin
        if N == 1:
            step1 = step
        cells = [plan.cells(s, N) for s in range(N)]
        line = {"config": cfg.name, "workload": cfg.description, "n_shards": N,
                "coarse_ms_max": max(coarse), "finish_ms": finish,
                "join_ms": joins, "join_ms_max": max(joins), "join_ms_mean": sum(joins) / N,
                "shard_cells_max_over_mean": max(cells) / (sum(cells) / N),
                "merge_ms_est": merge_est if N > 1 else 0.0, "finalize_ms": fin,
                "step_ms_pred": step, "cells_per_s_pred": cfg.cells() / (step * 1e-3),
                "efficiency_pred": step1 / (N * step) if step1 else None,
                "note": "phases timed per shard on one GPU; merge_ms_est from bytes at "
                        f"{NVLINK_MERGE_GBS:.0f} GB/s"}
        print(json.dumps(line), flush=True)
    plan.close()


if __name__ == "__main__":
    main()
