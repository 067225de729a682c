"""bench.py's launch contract: one JSON line from rank 0, other ranks exit 0.

The CPU test runs the reference arm (`--impl reference`, the oracle STOMP on a
bounded row sample) under torchrun with two ranks; the GPU test runs our arm
under torchrun with two ranks sharing cuda:0 over gloo (functional only: the
exchange is host-staged, no kernel waits on another rank's kernel), which
exercises the sharded prepare, the shard runs and the MIN merge of bench.py.
"""
import json
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


def _torchrun(nproc, args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.update(env_extra or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py")] + args
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_two_ranks_prints_one_line():
    r = _torchrun(2, ["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                      "--config", "C1", "--ref-seconds", "0.2"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["impl"] == "reference" and d["unit"] == "cells/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["config"] == "C1" and d["n_gpus"] == 2


@pytest.mark.gpu
def test_bench_two_ranks_gloo_on_one_gpu():
    r = _torchrun(2, ["--gpus", "2", "--steps", "1", "--warmup", "1", "--config", "C2",
                      "--no-cpu-baseline"], env_extra={"MPGPU_DIST_BACKEND": "gloo"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    # the run-time check of the multi-rank profile against rank 0's one-rank join
    assert d["multi_gpu_check"].startswith("bit-identical"), d["multi_gpu_check"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    # each rank evaluates about half of the cells
    assert 0.4 < d["roofline"]["cells_per_launch"] / d["config"]["cells_per_step"] < 0.6


@pytest.mark.gpu
def test_bench_two_ranks_separate_keys_check():
    r = _torchrun(2, ["--gpus", "2", "--steps", "1", "--warmup", "1", "--config", "C1",
                      "--no-cpu-baseline", "--no-e2e"],
                  env_extra={"MPGPU_DIST_BACKEND": "gloo", "MPGPU_SHARED_KEYS": "0"})
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_lines(r.stdout)[0]
    assert "NCCL MIN merge" in d["parallelism"]
    assert d["multi_gpu_check"].startswith("bit-identical"), d["multi_gpu_check"]


@pytest.mark.gpu
def test_bench_falls_back_when_the_shared_key_profile_mismatches():
    r = _torchrun(2, ["--gpus", "2", "--steps", "1", "--warmup", "1", "--config", "C1",
                      "--no-cpu-baseline"],
                  env_extra={"MPGPU_DIST_BACKEND": "gloo", "MPGPU_BENCH_FORCE_MISMATCH": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_lines(r.stdout)[0]
    assert "NCCL MIN merge" in d["parallelism"]
    assert "fell back" in d["multi_gpu_check"] and "matches bit for bit" in d["multi_gpu_check"]
    assert "NCCL" in d["e2e"]["api"] and d["e2e"]["value"] > 0
