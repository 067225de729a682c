"""Multi-GPU join: one process per GPU, diagonal shards, NCCL MIN merge.

Every rank holds the whole series, evaluates an equal-cell shard of the
diagonal work items (mpgpu_plan_run(shard=rank, n_shards=world)), and the
packed int64 keys are min-reduced across ranks — the join's only exchange
(SURVEY.md §8e), plus the same MIN over the small coarse-join keys inside the
sharded prepare (the warm start). Rank `root` then decodes the keys into the profile.
Shards never change the arithmetic of a cell, so the result is bit-identical
for any world size.
"""
from __future__ import annotations

from typing import Optional


def merge_keys_(row_keys, col_keys, group=None, root: Optional[int] = None) -> None:
    """In-place elementwise MIN of both key arrays across the group.

    root=None: all-reduce (every rank gets the merged keys); otherwise reduce
    to `root` only."""
    import torch.distributed as dist
    op = dist.ReduceOp.MIN
    host_staged = row_keys.is_cuda and dist.get_backend(group) == "gloo"
    for t in (row_keys, col_keys):
        if host_staged:
            # gloo (functional tests only: two ranks sharing one GPU) reduces host tensors
            h = t.cpu()
            dist.all_reduce(h, op=op, group=group)
            t.copy_(h)
        elif root is None:
            dist.all_reduce(t, op=op, group=group)
        else:
            dist.reduce(t, dst=root, op=op, group=group)


def sharded_prepare(plan, rank: int, world: int, group=None) -> None:
    """Prepare `plan` on every rank with the coarse warm start sharded too: each
    rank runs its shard of the coarse join, the coarse keys are all-reduced with
    MIN (every rank needs them), then each rank seeds its keys from them. The
    keys end up bit-identical to a single-rank prepare."""
    if world == 1:
        plan.prepare()
        return
    plan.prepare_shard(rank, world)
    ck = plan.coarse_keys()
    if ck is not None:
        merge_keys_(ck[0], ck[1], group=group, root=None)
    plan.prepare_finish()


def sharded_join(plan, rank: int, world: int, group=None, root: int = 0):
    """Run one rank's shard of `plan` (a paper_1904_12626_b200.Plan) and merge.

    Returns the MatrixProfile device arrays on `root`, None elsewhere."""
    sharded_prepare(plan, rank, world, group=group)
    plan.run(rank, world)
    if world > 1:
        rk, ck = plan.keys()
        merge_keys_(rk, ck, group=group, root=root)
    if rank == root:
        return plan.outputs()
    return None
