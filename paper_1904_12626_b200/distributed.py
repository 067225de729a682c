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


def _check_peer_atomics(device: int, rank: int, world: int, group) -> str:
    """'' when this GPU has native peer atomics to every other rank's GPU, else
    why not (collective: gathers every rank's PCI bus id)."""
    import torch.distributed as dist
    import paper_1904_12626_b200 as mp
    L = mp.lib()
    buf = ctypes.create_string_buffer(64)
    bus = buf.value.decode() if L.mpgpu_device_pci_bus_id(device, buf, 64) == 0 else ""
    buses = [None] * world
    dist.all_gather_object(buses, bus, group=group)
    assume = os.environ.get("MPGPU_ASSUME_PEER_ATOMICS", "0") == "1"
    for r, b in enumerate(buses):
        if r == rank:
            continue
        a = L.mpgpu_peer_atomics(device, b.encode()) if b else -1
        if a == 0 or (a < 0 and not assume):
            return f"no verified native peer atomics between this GPU and rank {r}'s ({b or '?'})"
    return ""


class Region:
    """A device region mapped at one contiguous address in every rank, whose
    2 MB chunks live on the ranks `owners` names (mpgpu_stripes_*): chunk fds
    go to every other rank over SCM_RIGHTS, every rank imports and maps all of
    them. Collective; on failure every rank raises at the same point.
    `prepared` lets the caller do work on the mapping before the final
    agreement (e.g. attach a plan) so that its failure is agreed on too."""

    def __init__(self, nbytes: int, owners, rank: int, world: int, device, device_index: int,
                 group=None, why: str = "", prepared=None):
        import paper_1904_12626_b200 as mp
        L = mp.lib()
        self._s = None
        self.base = 0
        self.nbytes = int(nbytes)
        my_fds = {}
        if not why:
            own_arr = (ctypes.c_int32 * max(1, len(owners)))(*owners)
            s = L.mpgpu_stripes_create(self.nbytes, world, rank, device_index, own_arr)
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
        if not _agree(not why, device, group):
            _close_fds(my_fds)
            self.close()
            raise RuntimeError(why or "striped region unavailable on another rank")
        try:
            got = exchange_fds(my_fds, rank, world, group=group)
        finally:
            _close_fds(my_fds)
        try:
            for c, fd in sorted(got.items()):
                mp._check(L.mpgpu_stripes_import_fd(self._s, c, fd))
            base = ctypes.c_void_p()
            mp._check(L.mpgpu_stripes_map(self._s, ctypes.byref(base)))
            self.base = base.value
            if prepared is not None:
                prepared(self)
            why = ""
        except Exception as e:  # noqa: BLE001 -- agreed on collectively below
            why = str(e)
        finally:
            _close_fds(got)
        if not _agree(not why, device, group):
            self.close()
            raise RuntimeError(why or "striped region unavailable on another rank")
        self.chunks = int(L.mpgpu_stripes_num_chunks(self._s))
        self.chunk_bytes = int(L.mpgpu_stripes_chunk_bytes(self._s))

    def close(self) -> None:
        import paper_1904_12626_b200 as mp
        if self._s is not None:
            mp.lib().mpgpu_stripes_destroy(self._s)
            self._s = None
            self.base = 0


def _close_fds(fds: dict) -> None:
    for fd in fds.values():
        try:
            os.close(fd)
        except OSError:
            pass
    fds.clear()


def _align(n: int, a: int = 256) -> int:
    return (n + a - 1) // a * a


class SharedKeys:
    """The join's keys in one region striped over every rank's HBM, and the
    profile in a region on the root that every rank writes its rows of.

    Keys: chunk c of the region (the VMM granularity, 2 MB) lives on the rank
    that mpgpu_plan_key_region_owners picks (chunks dealt by modelled key
    traffic, largest first to the least-loaded rank). Every rank maps all
    chunks into one contiguous range and attaches its plan (fine and coarse
    warm-start keys), so every rank's k_join reads thresholds from and RED.MINs
    into the same keys while it computes: the min-merge is fused into the join,
    each shard filters against the whole job's best-so-far (about the one-GPU
    replay rate), and the key traffic spreads over all GPUs' NVLink ports
    instead of converging on one owner. Rank `root` owns the
    keys' contents: it resets and warm-starts them.

    Profile: every chunk on the root; after the join each rank decodes its
    1/world of the rows (mpgpu_plan_finalize_shard) straight into it over
    NVLink, so the finalize is sharded too and no gather follows.

    Requires native peer atomics between every pair of ranks' GPUs (NVLink;
    checked here, MPGPU_ASSUME_PEER_ATOMICS=1 skips the check when a peer GPU is
    not visible to this process). Collective use only (every rank constructs
    it); on failure every rank raises at the same point."""

    def __init__(self, plan, rank: int, world: int, group=None, root: int = 0):
        import torch.distributed as dist
        import paper_1904_12626_b200 as mp
        L = mp.lib()
        self.plan, self.rank, self.world, self.root, self.group = plan, rank, world, root, group
        self.keys = self.out = None
        self.attached = False
        dev = plan.a.device
        why = _check_peer_atomics(plan.device, rank, world, group)
        nbytes, owners, self.max_share = 0, [], 0.0
        if not why:
            gran = int(L.mpgpu_stripes_granularity(plan.device))
            if gran <= 0:
                why = "no CUDA VMM: " + L.mpgpu_last_error().decode(errors="replace")
            else:
                nbytes = plan.key_region_bytes()
                owners, self.max_share = plan.key_region_owners(gran, world)

        def attach(region):
            plan.attach_key_region(region.base, nbytes, owner=rank == root)
            self.attached = True
            if rank == root:
                plan.reset_keys()  # the first join starts from empty keys
            plan.stream.synchronize()

        try:
            self.keys = Region(nbytes, owners, rank, world, dev, plan.device, group, why, attach)
            # the profile, all on the root: mp_a, pi_a, then left/right (self) or mp_b/pi_b (AB)
            La, Lb = plan.La, plan.Lb
            lens = [La, La, La, La] if plan.self_join else [La, La, Lb, Lb]
            self._out_off = [0]
            for n in lens:
                self._out_off.append(self._out_off[-1] + _align(8 * n))
            gran = self.keys.chunk_bytes
            n_out = (self._out_off[-1] + gran - 1) // gran
            self.out = Region(self._out_off[-1], [root] * n_out, rank, world, dev, plan.device, group)
        except Exception:
            self.close()
            raise
        dist.barrier(group=group)  # the owner's reset is visible before anyone seeds
        self.chunks, self.chunk_bytes = self.keys.chunks, self.keys.chunk_bytes
        self.coarse_shared = True
        plan._coarse_shared = True

    def output_views(self):
        """The profile arrays in the root's output region, as CUDA tensors on this
        rank (the root's are local memory). Valid until the next join."""
        import torch
        import paper_1904_12626_b200 as mp
        dev = torch.device("cuda", self.plan.device)
        names = (["mp_a", "pi_a", "left_a", "right_a"] if self.plan.self_join
                 else ["mp_a", "pi_a", "mp_b", "pi_b"])
        lens = [self.plan.La] * 4 if self.plan.self_join else [self.plan.La] * 2 + [self.plan.Lb] * 2
        out = {}
        for k, (name, n) in enumerate(zip(names, lens)):
            typ = "<f8" if name.startswith("mp") else "<i8"
            out[name] = torch.as_tensor(mp._CudaArray(self.out.base + self._out_off[k], n, typ, self),
                                        device=dev)
        return out

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
        """Detach the plan (back to its own keys) and release the regions."""
        if self.attached:
            try:
                self.plan.stream.synchronize()
                self.plan.attach_key_region(0, 0, False)
            finally:
                self.attached = False
                self.plan._coarse_shared = self.coarse_shared = False
        for r in (self.out, self.keys):
            if r is not None:
                r.close()
        self.out = self.keys = None


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


def shared_outputs(plan, rank: int, root: int = 0, shared=None, group=None):
    """Decode the shared keys into the profile, then let the root empty them for
    the next join. With `shared` (a SharedKeys) every rank decodes its 1/world of
    the rows straight into the root's output region (collective; a barrier
    follows, then the root resets the keys); without it the root decodes alone.
    Returns the profile arrays on the root (with `shared`: views of its output
    region, valid until the next join), None elsewhere."""
    if shared is not None and shared.out is not None:
        import torch.distributed as dist
        world = shared.world
        o = shared.output_views()
        if plan.self_join:
            plan.finalize_shard(rank, world, o["mp_a"], o["pi_a"], o["left_a"], o["right_a"])
        else:
            plan.finalize_shard(rank, world, o["mp_a"], o["pi_a"], mp_b=o["mp_b"], pi_b=o["pi_b"])
        plan.stream.synchronize()
        dist.barrier(group=group)  # every rank's rows have landed and nobody reads the keys
        if rank != root:
            return None
        plan.reset_keys()
        return o
    if rank != root:
        return None
    out = plan.outputs()
    plan.reset_keys()
    return out


def shared_keys_join(plan, rank: int, world: int, group=None, root: int = 0, shared=None):
    """One join over keys shared through SharedKeys (attached beforehand):
    shared_prepare, this rank's shard of the join straight into the shared
    keys, shared_finish, then the profile is decoded (every rank its rows into
    the root's output region when `shared` is given, else the root alone).
    Returns the MatrixProfile device arrays on the root, None elsewhere."""
    shared_prepare(plan, rank, world, group=group, root=root)
    plan.run(rank, world)
    shared_finish(plan, group=group)
    return shared_outputs(plan, rank, root=root, shared=shared, group=group)
