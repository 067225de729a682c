"""The N>1 path on CPU: diagonal shards per rank, packed-key MIN merge over
torch.distributed (gloo, world_size 2), decode, compare with the oracle.

The per-rank cell evaluation here is a numpy model of the device kernel's
key production (exact correlations, keys.pack); what is under test is the
sharding rule, the key format and the collective merge that bench.py and
paper_1904_12626_b200.distributed drive over NCCL on GPUs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_1904_12626_b200 import distributed, keys
from tests.parity import exact_dist

W, EZ, N = 24, 0.5, 700
BAND = 8  # diagonals per work band in this model


def _series():
    return np.cumsum(np.random.Generator(np.random.MT19937(77)).standard_normal(N))


def _shard_keys(x, rank, world):
    """Row (right) and column (left) keys of this rank's diagonal bands."""
    win = np.lib.stride_tricks.sliding_window_view(x, W)
    mu = win.mean(1)
    sd = win.std(1)
    z = (win - mu[:, None]) / sd[:, None]
    L = z.shape[0]
    zone = int(np.floor(W * EZ + 0.5))
    bits = keys.index_bits(L)
    row = np.full(L, keys.KEY_NONE, np.int64)
    col = np.full(L, keys.KEY_NONE, np.int64)
    for k in range(zone + 1, L):
        if ((k - zone - 1) // BAND) % world != rank:
            continue
        i = np.arange(0, L - k)
        j = i + k
        c = np.einsum("ij,ij->i", z[i], z[j]) / W
        row[i] = np.minimum(row[i], keys.pack(c, j, bits))
        col[j] = np.minimum(col[j], keys.pack(c, i, bits))
    return row, col, bits


def _worker(rank, world, port, x, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    row, col, _ = _shard_keys(x, rank, world)
    rt, ct = torch.from_numpy(row.copy()), torch.from_numpy(col.copy())
    distributed.merge_keys_(rt, ct)
    if rank == 0:
        out_q.put((rt.numpy().copy(), ct.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_merge_matches_oracle(oracle_lib):
    x = _series()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, q)) for r in range(2)]
    for p in procs:
        p.start()
    row, col = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the 2-rank merge equals the single-rank keys exactly (shard invariance)
    row1, col1, bits = _shard_keys(x, 0, 1)
    assert np.array_equal(row, row1) and np.array_equal(col, col1)
    # decode: PI = smaller of left/right keys (ties -> smaller index, i.e. left)
    _, ridx = keys.unpack(row, bits)
    _, lidx = keys.unpack(col, bits)
    best = np.minimum(row, col)
    _, pidx = keys.unpack(best, bits)
    ref = oracle_lib.brute_force_mp(x, None, W, EZ)
    L = ref[0].size
    mp = np.array([exact_dist(x, i, x, int(pidx[i]), W) if pidx[i] >= 0 else np.inf for i in range(L)])
    fin = np.isfinite(ref[0])
    assert np.array_equal(np.isfinite(mp), fin)
    assert np.max(np.abs(mp[fin] - ref[0][fin])) < 1e-8
    assert np.array_equal(pidx, ref[1]) and np.array_equal(lidx, ref[2]) and np.array_equal(ridx, ref[3])


def test_world_size_invariance_model():
    """Keys from 1, 2, 3 and 4 shards min-merge to the same array."""
    x = _series()
    base = _shard_keys(x, 0, 1)
    for world in (2, 3, 4):
        parts = [_shard_keys(x, r, world) for r in range(world)]
        row = np.minimum.reduce([p[0] for p in parts])
        col = np.minimum.reduce([p[1] for p in parts])
        assert np.array_equal(row, base[0]) and np.array_equal(col, base[1])


class _FakePlan:
    """Stands in for a Plan on a machine without a GPU: the C ABI can neither
    verify native peer atomics nor create the striped region, and SharedKeys
    must not leave the other ranks waiting."""

    device = 0

    class a:  # noqa: N801 -- mirrors Plan.a.device
        device = torch.device("cpu")

    def key_region_bytes(self):
        return 1 << 22

    def reset_keys(self):
        raise AssertionError("not reached: the region is never created")


def _fallback_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sk = distributed.SharedKeys.try_create(_FakePlan(), rank, world)
    out_q.put((rank, sk is None))
    dist.barrier()
    dist.destroy_process_group()


def test_shared_keys_fall_back_together_when_region_fails():
    """Every rank gets None (and so keeps the NCCL merge) when the striped key
    region cannot be set up; nobody hangs in the fd exchange."""
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: True, 1: True}


def _fd_worker(rank, world, port, n_chunks, out_q):
    """Each rank 'owns' chunks c % world == rank, each an anonymous file
    holding (rank, chunk); after the exchange every rank reads the files it
    received and reports which chunks came from whom."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = {}
    for c in range(rank, n_chunks, world):
        fd = os.memfd_create(f"chunk{c}")
        os.write(fd, f"{rank}:{c}".encode())
        mine[c] = fd
    got = distributed.exchange_fds(dict(mine), rank, world)
    seen = {}
    for c, fd in got.items():
        seen[c] = os.pread(fd, 64, 0).decode()
        os.close(fd)
    for fd in mine.values():
        os.close(fd)
    out_q.put((rank, seen))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_chunks", [(2, 5), (3, 7), (2, 450)])
def test_exchange_fds_world(world, n_chunks):
    """The SCM_RIGHTS exchange behind the striped key region (more than one
    message per peer at 450 chunks): every rank ends up with a working fd for
    every chunk the other ranks own, and none of its own."""
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fd_worker, args=(r, world, port, n_chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        want = {c: f"{c % world}:{c}" for c in range(n_chunks) if c % world != r}
        assert got[r] == want
