"""Multi-GPU join: one process per GPU, diagonal shards, keys shared or MIN-merged.

Every rank holds the whole series and evaluates an equal-cell shard of the
diagonal work items (mpgpu_plan_run(shard=rank, n_shards=world)). The join's
only exchange is the element-wise MIN of the packed int64 (score, index) keys
(the reference's worker merge, profile.hpp:66-68):

* default (SharedKeys): the keys live in one region striped over every rank's
  HBM (2 MB chunks round-robin, CUDA VMM) and mapped into every process; each
  rank's k_join reads its thresholds from and RED.MINs its candidates into it
  while it computes, so the merge is fused into the join and no single GPU
  serves every other rank's key traffic;
* fallback (sharded_join): separate keys per rank, MIN-reduced with NCCL after
  the join.

Shards never change the arithmetic of a cell, so the result is bit-identical
for any world size and either exchange.
"""
from __future__ import annotations

import ctypes
import json
import os
import secrets
import socket
import struct
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


def _agree(ok: bool, device, group) -> bool:
    """True on every rank iff `ok` on every rank (a collective)."""
    import torch
    import torch.distributed as dist
    dev = device if dist.get_backend(group) == "nccl" else "cpu"
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return int(flag.item()) == 1


_FDS_PER_MSG = 200  # below the kernel's SCM_MAX_FD (253)


def exchange_fds(my_fds: dict, rank: int, world: int, group=None, timeout: float = 120.0) -> dict:
    """Send this rank's {chunk: fd} to every other rank and receive theirs, over
    abstract-namespace Unix sockets with SCM_RIGHTS (one process per GPU on one
    node). Returns {chunk: fd} of every other rank's chunks (received copies;
    the caller closes them). Collective."""
    import torch.distributed as dist
    token = [secrets.token_hex(8) if rank == 0 else None]
    dist.broadcast_object_list(token, src=0, group=group)
    name = lambda r: f"\0mpgpu-stripes-{token[0]}-{r}"  # noqa: E731
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_SEQPACKET)
    srv.bind(name(rank))
    srv.listen(max(1, world))
    srv.settimeout(timeout)
    got = {}
    try:
        dist.barrier(group=group)  # every listener is up
        chunks = sorted(my_fds)
        for peer in range(world):
            if peer == rank:
                continue
            c = socket.socket(socket.AF_UNIX, socket.SOCK_SEQPACKET)
            c.settimeout(timeout)
            c.connect(name(peer))
            for q in range(0, max(1, len(chunks)), _FDS_PER_MSG):
                part = chunks[q:q + _FDS_PER_MSG]
                body = json.dumps({"rank": rank, "chunks": part}).encode()
                socket.send_fds(c, [struct.pack("<I", len(body)) + body], [my_fds[k] for k in part])
            c.sendall(b"\0\0\0\0")  # end of this rank's chunks
            c.close()
        for _ in range(world - 1):
            conn, _ = srv.accept()
            conn.settimeout(timeout)
            with conn:
                while True:
                    msg, fds, _flags, _addr = socket.recv_fds(conn, 1 << 16, _FDS_PER_MSG)
                    (blen,) = struct.unpack("<I", msg[:4])
                    if blen == 0:
                        break
                    meta = json.loads(msg[4:4 + blen])
                    if len(fds) != len(meta["chunks"]):
                        raise RuntimeError("striped keys: lost file descriptors in transit")
                    got.update(zip(meta["chunks"], fds))
    finally:
        srv.close()
    return got


class SharedKeys:
    """The join's keys in one region striped over every rank's HBM.

    Chunk c of the region (the VMM granularity, 2 MB) lives on the rank that
    mpgpu_plan_key_region_owners picks: chunks are dealt by modelled key
    traffic, largest first to the least-loaded rank.
    Every rank maps all chunks into one contiguous range and attaches its plan
    (fine and coarse warm-start keys), so every rank's k_join reads thresholds
    from and RED.MINs into the same keys while it computes: the min-merge is
    fused into the join, each shard filters against the whole job's
    best-so-far (about the one-GPU replay rate), and the key traffic spreads
    over all GPUs' NVLink ports instead of converging on one owner
    (DESIGN.md §7). Rank `root` owns the keys' contents: it resets and
    warm-starts them.

    Requires native peer atomics between every pair of ranks' GPUs (NVLink;
    checked here, MPGPU_ASSUME_PEER_ATOMICS=1 skips the check when a peer GPU is
    not visible to this process). Collective use only (every rank constructs
    it); on failure every rank raises at the same point."""

    def __init__(self, plan, rank: int, world: int, group=None, root: int = 0):
        import torch.distributed as dist
        import paper_1904_12626_b200 as mp
        L = mp.lib()
        self.plan, self.rank, self.world, self.root, self.group = plan, rank, world, root, group
        self._s = None
        self.attached = False
        dev = plan.a.device
        # 1) native peer atomics to every other rank's GPU
        buf = ctypes.create_string_buffer(64)
        bus = buf.value.decode() if L.mpgpu_device_pci_bus_id(plan.device, buf, 64) == 0 else ""
        buses = [None] * world
        dist.all_gather_object(buses, bus, group=group)
        assume = os.environ.get("MPGPU_ASSUME_PEER_ATOMICS", "0") == "1"
        why = ""
        for r, b in enumerate(buses):
            if r == rank:
                continue
            a = L.mpgpu_peer_atomics(plan.device, b.encode()) if b else -1
            if a == 0 or (a < 0 and not assume):
                why = f"no verified native peer atomics between this GPU and rank {r}'s ({b or '?'})"
                break
        # 2) this rank's chunks, exported as fds
        nbytes = 0
        my_fds = {}
        if not why:
            nbytes = plan.key_region_bytes()
            gran = L.mpgpu_stripes_granularity(plan.device)
            owners, self.max_share = plan.key_region_owners(gran, world) if gran > 0 else ([], 0.0)
            own_arr = (ctypes.c_int32 * max(1, len(owners)))(*owners)
            s = L.mpgpu_stripes_create(nbytes, world, rank, plan.device, own_arr) if gran > 0 else None
            if not s:
                why = "striped region: " + L.mpgpu_last_error().decode(errors="replace")
            else:
                self._s = ctypes.c_void_p(s)
                for c in range(L.mpgpu_stripes_num_chunks(self._s)):
                    if L.mpgpu_stripes_owner(self._s, c) != rank:
                        continue
                    fd = L.mpgpu_stripes_export_fd(self._s, c)
                    if fd < 0:
                        why = "export: " + L.mpgpu_last_error().decode(errors="replace")
                        break
                    my_fds[c] = fd
        if not _agree(not why, dev, group):
            self._close_fds(my_fds)
            self.close()
            raise RuntimeError(why or "striped keys unavailable on another rank")
        # 3) exchange, import, map, attach
        try:
            got = exchange_fds(my_fds, rank, world, group=group)
        finally:
            self._close_fds(my_fds)
        try:
            for c, fd in sorted(got.items()):
                mp._check(L.mpgpu_stripes_import_fd(self._s, c, fd))
            base = ctypes.c_void_p()
            mp._check(L.mpgpu_stripes_map(self._s, ctypes.byref(base)))
            plan.attach_key_region(base.value, nbytes, owner=rank == root)
            self.attached = True
            if rank == root:
                plan.reset_keys()  # the first join starts from empty keys
            plan.stream.synchronize()
            why = ""
        except Exception as e:  # noqa: BLE001 -- agreed on collectively below
            why = str(e)
        finally:
            self._close_fds(got)
        if not _agree(not why, dev, group):
            self.close()
            raise RuntimeError(why or "striped keys unavailable on another rank")
        dist.barrier(group=group)  # the owner's reset is visible before anyone seeds
        self.chunks = int(L.mpgpu_stripes_num_chunks(self._s))
        self.chunk_bytes = int(L.mpgpu_stripes_chunk_bytes(self._s))
        self.coarse_shared = True
        plan._coarse_shared = True

    @staticmethod
    def _close_fds(fds: dict) -> None:
        for fd in fds.values():
            try:
                os.close(fd)
            except OSError:
                pass
        fds.clear()

    @classmethod
    def try_create(cls, plan, rank: int, world: int, group=None, root: int = 0):
        """SharedKeys, or None on every rank when any rank cannot map the region
        (no VMM, no native peer atomics): the caller then keeps separate keys
        and MIN-reduces them after the join."""
        import sys
        import torch.distributed as dist
        sk, ok = None, True
        try:
            sk = cls(plan, rank, world, group=group, root=root)
        except Exception as e:  # noqa: BLE001 -- reported, then agreed on collectively
            ok = False
            print(f"[mprof_b200] rank {rank}: shared keys unavailable ({e}); using the NCCL merge",
                  file=sys.stderr)
        dev = plan.a.device if dist.get_backend(group) == "nccl" else "cpu"
        if not _agree(ok, dev, group):
            if sk is not None:
                sk.close()
            return None
        return sk

    def close(self) -> None:
        """Detach the plan (back to its own keys) and release the region."""
        import paper_1904_12626_b200 as mp
        if self.attached:
            try:
                self.plan.stream.synchronize()
                self.plan.attach_key_region(0, 0, False)
            finally:
                self.attached = False
                self.plan._coarse_shared = self.coarse_shared = False
        if self._s is not None:
            mp.lib().mpgpu_stripes_destroy(self._s)
            self._s = None


def shared_prepare(plan, rank: int, world: int, group=None, root: int = 0) -> None:
    """Warm start over shared keys, sharded: every rank runs stats (the owner
    also resets and warm-starts the coarse keys); after a barrier every rank
    runs its shard of the coarse join into the shared coarse keys; after a
    second barrier every rank RED.MINs its share of the warm-start cells into
    the shared keys and may start its join at once. Each barrier follows a
    synchronize of the plan's stream, so the owner's reset of the fine keys
    (shared_outputs of the previous join) and its coarse-key reset have landed
    before any rank writes into them."""
    import torch.distributed as dist
    plan.prepare_shared(rank, world)
    plan.stream.synchronize()
    dist.barrier(group=group)
    if getattr(plan, "_coarse_shared", False):
        plan.coarse_run(rank, world)
        plan.stream.synchronize()
        dist.barrier(group=group)
    plan.seed_shared(rank, world)


def shared_finish(plan, group=None) -> None:
    """Wait until every rank's join has landed in the shared keys."""
    import torch.distributed as dist
    plan.stream.synchronize()
    dist.barrier(group=group)


def shared_outputs(plan, rank: int, root: int = 0):
    """The root decodes the shared keys, then empties them for the next join
    (on its stream; the next shared_prepare synchronizes it before its barrier)."""
    if rank != root:
        return None
    out = plan.outputs()
    plan.reset_keys()
    return out


def shared_keys_join(plan, rank: int, world: int, group=None, root: int = 0):
    """One join over keys shared through SharedKeys (attached beforehand):
    shared_prepare, this rank's shard of the join straight into the shared
    keys, shared_finish, then the root decodes the keys.
    Returns the MatrixProfile device arrays on the root, None elsewhere."""
    shared_prepare(plan, rank, world, group=group, root=root)
    plan.run(rank, world)
    shared_finish(plan, group=group)
    return shared_outputs(plan, rank, root=root)
