"""Multi-process join with keys shared over CUDA IPC (bench.py's N > 1 path):
two and three ranks, all on cuda:0 (functional only; a real run has one GPU
per rank and the mappings go over NVLink). The profile must be bit-identical
to a one-process join: cells never change arithmetic with sharding, and the
shared keys are the exact MIN of every rank's candidates."""
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
                                            (2, 1 << 14, 100, "ab")])
def test_shared_keys_join_matches_single_process(nproc, n, m, kind):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_shared_keys_worker.py"), str(n), str(m), kind]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "OK" in r.stdout
