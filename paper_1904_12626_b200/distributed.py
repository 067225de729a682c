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

import ctypes
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


class SharedKeys:
    """Rank `root`'s key arrays mapped into every rank's plan over CUDA IPC.

    One process per GPU: the root exports its two key allocations as IPC
    handles, the other ranks open them (peer-memory mappings over NVLink) and
    attach their plans. Every rank's k_join then reads its filter thresholds
    from, and RED.MINs its candidates into, the same keys while it computes:
    the min-merge is fused into the join (no reduce afterwards), and each
    shard filters against the whole job's best-so-far instead of only its
    own, so it replays about as few blocks as a one-GPU run.
    Collective use only (every rank constructs it)."""

    def __init__(self, plan, rank: int, world: int, group=None, root: int = 0):
        import torch.distributed as dist
        import paper_1904_12626_b200 as mp
        self.plan, self.rank, self.root, self.group = plan, rank, root, group
        self.opened = []
        handles = [None]
        if rank == root:
            try:
                hs = []
                cr, cc = plan.coarse_key_ptrs()  # the coarse warm-start keys are shared too
                for ptr in plan.key_ptrs() + ((cr, cc) if cr else ()):
                    buf = (ctypes.c_char * 64)()
                    mp._check(mp.lib().mpgpu_ipc_export(ctypes.c_void_p(ptr), buf, plan.device))
                    hs.append(bytes(buf))
                plan.reset_keys()  # the first join starts from empty keys
                plan.stream.synchronize()
                handles = [hs]
            except Exception as e:  # noqa: BLE001 -- tell the other ranks before raising
                handles = [f"export failed: {e}"]
                try:
                    plan.attach_coarse_key_ptrs(0, 0)  # back to a per-rank coarse phase
                except Exception:  # noqa: BLE001
                    pass
        dist.broadcast_object_list(handles, src=root, group=group)
        if isinstance(handles[0], str):
            raise RuntimeError(handles[0])
        if rank != root:
            ptrs = []
            for h in handles[0]:
                p = ctypes.c_void_p()
                mp._check(mp.lib().mpgpu_ipc_open(h, ctypes.byref(p), plan.device))
                self.opened.append(p.value)
                ptrs.append(p.value)
            plan.attach_key_ptrs(ptrs[0], ptrs[1])
            if len(ptrs) == 4:
                plan.attach_coarse_key_ptrs(ptrs[2], ptrs[3])
        self.coarse_shared = len(handles[0]) == 4
        plan._coarse_shared = self.coarse_shared

    @classmethod
    def try_create(cls, plan, rank: int, world: int, group=None, root: int = 0):
        """SharedKeys, or None on every rank when any rank cannot map the keys
        (e.g. no peer access between its GPU and the root's): the caller then
        keeps separate keys and MIN-reduces them after the join."""
        import sys
        import torch
        import torch.distributed as dist
        sk, ok = None, 1
        try:
            sk = cls(plan, rank, world, group=group, root=root)
        except Exception as e:  # noqa: BLE001 -- reported, then agreed on collectively
            ok = 0
            print(f"[mprof_b200] rank {rank}: shared keys unavailable ({e}); using the NCCL merge",
                  file=sys.stderr)
        flag = torch.tensor([ok], dtype=torch.int32,
                            device=plan.a.device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()) == 0:
            if sk is not None:
                sk.close()
            return None
        return sk

    def close(self) -> None:
        import paper_1904_12626_b200 as mp
        if getattr(self, "coarse_shared", False):
            self.plan.attach_coarse_key_ptrs(0, 0)  # every rank back to its own coarse keys
            self.plan._coarse_shared = self.coarse_shared = False
        if self.opened:
            self.plan.attach_key_ptrs(0, 0)
            for p in self.opened:
                mp.lib().mpgpu_ipc_close(ctypes.c_void_p(p), self.plan.device)
            self.opened = []


def shared_prepare(plan, rank: int, world: int, stream, group=None, root: int = 0) -> None:
    """Warm start over shared keys, sharded: every rank runs stats and its
    shard of the coarse join, the coarse keys are MIN-all-reduced, then every
    rank RED.MINs its share of the warm-start cells into the shared keys. No
    barrier before the join: the keys only tighten the filter, and the owner
    reset them before the previous join's end barrier released anyone. Without
    a coarse phase (small joins) a barrier orders the ranks after that reset."""
    import torch.distributed as dist
    plan.prepare_shared(rank, world)
    if getattr(plan, "_coarse_shared", False):
        # shared coarse keys: the owner's coarse prepare (reset + its warm start)
        # lands before any rank's coarse shard, and every shard before the seeding
        stream.synchronize()
        dist.barrier(group=group)
        plan.coarse_run(rank, world)
        stream.synchronize()
        dist.barrier(group=group)
    else:
        ck = plan.coarse_keys()
        if ck is not None:
            merge_keys_(ck[0], ck[1], group=group, root=None)
        else:
            dist.barrier(group=group)
    plan.seed_shared(rank, world)


def shared_finish(stream, group=None) -> None:
    """Wait until every rank's join has landed in the shared keys."""
    import torch.distributed as dist
    stream.synchronize()
    dist.barrier(group=group)


def shared_outputs(plan, rank: int, root: int = 0):
    """The root decodes the shared keys, then empties them for the next join
    (before any rank can pass the next join's coarse all-reduce)."""
    if rank != root:
        return None
    out = plan.outputs()
    plan.reset_keys()
    return out


def shared_keys_join(plan, rank: int, world: int, stream, group=None, root: int = 0):
    """One join over keys shared through SharedKeys (attached beforehand):
    shared_prepare, this rank's shard of the join straight into the shared
    keys, shared_finish, then the root decodes the keys.
    Returns the MatrixProfile device arrays on the root, None elsewhere."""
    shared_prepare(plan, rank, world, stream, group=group, root=root)
    plan.run(rank, world)
    shared_finish(stream, group=group)
    return shared_outputs(plan, rank, root=root)
