"""Multi-process join with the keys in one region striped over the ranks'
GPUs (bench.py's N > 1 path): two and three ranks, all on cuda:0 (functional
only; a real run has one GPU per rank and the chunk mappings go over NVLink).
The profile must be bit-identical to a one-process join: cells never change
arithmetic with sharding, and the shared keys are the exact MIN of every
rank's candidates. n = 2^19 makes the warm start's rows per thread > 1 on one
rank, where an earlier build sized them from the shard's share (the seed
points then moved with the world size). Eight ranks at n = 2^17 have fewer
2 MB chunks than ranks: most ranks own no chunk and map the others' only."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("nproc,n,m,kind", [(2, 1 << 16, 128, "self"), (3, 1 << 14, 64, "self"),
                                            (2, 1 << 14, 100, "ab"), (2, 1 << 19, 128, "self"),
                                            (3, 1 << 18, 200, "ab"), (8, 1 << 17, 128, "self")])
def test_shared_keys_join_matches_single_process(nproc, n, m, kind):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_shared_keys_worker.py"), str(n), str(m), kind]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


@pytest.mark.gpu
def test_key_region_owner_table():
    """The striped region's chunk owners (mpgpu_plan_key_region_owners): every
    chunk has an owner, every rank owns a chunk when there are enough, the
    busiest rank's modelled share of the key reads is at least 1/N and, at
    C5-like sizes, close to it."""
    import numpy as np
    import torch
    import paper_1904_12626_b200 as mp
    x = torch.from_numpy(np.cumsum(np.random.default_rng(3).standard_normal(1 << 21))).cuda()
    plan = mp.Plan(x, None, 128, 64)
    gran = int(mp.lib().mpgpu_stripes_granularity(plan.device))
    assert gran >= 1 << 21
    nbytes = plan.key_region_bytes()
    for n in (1, 2, 3, 8):
        owners, share = plan.key_region_owners(gran, n)
        assert len(owners) == -(-nbytes // gran)
        assert all(0 <= o < n for o in owners)
        if len(owners) >= n:
            assert set(owners) == set(range(n))
        assert 1.0 / n - 1e-9 <= share <= 1.0
    owners, share = plan.key_region_owners(gran, 2)
    assert share < 0.55  # 2^21 windows: 33 chunks balance to ~1/2
    plan.close()
