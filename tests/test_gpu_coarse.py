"""The coarse warm start (K2b) on small inputs: forced on with MPGPU_COARSE_MIN=0
in a subprocess (the env is read once per process), the join must still match
brute force on self-joins, AB-joins, flat runs and near-constant series."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import json, sys
import numpy as np
sys.path.insert(0, ROOT)
import oracle
import paper_1904_12626_b200 as mp
from tests.parity import close, index_mismatches
oracle.build()
g = np.random.default_rng(77)
fails = []
cases = []
for t in range(12):
    n = int(g.integers(800, 4000)); w = int(g.choice([32, 48, 64, 100, 128]))
    x = np.cumsum(g.standard_normal(n))
    if t % 4 == 1:
        x[n // 3: n // 3 + 2 * w] = x[n // 3]          # flat run
    if t % 4 == 2:
        x = np.sin(np.arange(n) * 2 * np.pi / 50.0) + 1e-2 * g.standard_normal(n)
    cases.append((x, None, w, (0.0, 0.25, 0.5)[t % 3]))
for t in range(4):
    a = np.cumsum(g.standard_normal(int(g.integers(600, 3000))))
    b = np.cumsum(g.standard_normal(int(g.integers(600, 3000))))
    cases.append((a, b, 64, 0.0))
for ci, (a, b, w, ez) in enumerate(cases):
    if b is None:
        r = mp.stomp(a, None, w, ez)
        ref = oracle.brute_force_mp(a, None, w, ez)
        ok = close(r.values, ref[0])[0]
        rows = np.arange(r.size())
        bad = (index_mismatches(r.index, ref[1], rows, a, a, w) +
               index_mismatches(r.left_index, ref[2], rows, a, a, w) +
               index_mismatches(r.right_index, ref[3], rows, a, a, w))
    else:
        pa, pb = mp.stomp_ab(a, b, w)
        ra = oracle.brute_force_mp(a, b, w); rb = oracle.brute_force_mp(b, a, w)
        ok = close(pa.values, ra[0])[0] and close(pb.values, rb[0])[0]
        bad = (index_mismatches(pa.index, ra[1], np.arange(pa.size()), a, b, w) +
               index_mismatches(pb.index, rb[1], np.arange(pb.size()), b, a, w))
    if not ok or bad:
        fails.append((ci, bool(ok), len(bad)))
import torch
x = torch.from_numpy(np.cumsum(g.standard_normal(3000))).cuda()
plan = mp.Plan(x, None, 64, 32)
plan.prepare()
torch.cuda.synchronize()
print(json.dumps({"cases": len(cases), "fails": fails, "prepare_launches": plan.launches()}))
'''


def test_coarse_forced_matches_brute_force():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MPGPU_COARSE_MIN="0")
    out = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + SCRIPT], env=env,
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["cases"] == 16 and res["fails"] == [], res
    # stats (1) + key fill (2) + spread init (1) alone would be 4: the coarse
    # phase adds the PAA, the nested plan's prepare (4) + join (1) and two
    # exploit launches
    assert res["prepare_launches"] >= 4 + 1 + 5 + 2, res


def test_sharded_prepare_bit_identical():
    """Virtual ranks on one GPU: every rank prepares its shard of the coarse
    join, the coarse keys are min-merged, each rank runs its shard of the join,
    and the min-merged result equals a single-rank join bit for bit."""
    import numpy as np
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_12626_b200 as mp
    x = torch.from_numpy(np.cumsum(np.random.default_rng(31).standard_normal(52000))).cuda()
    w, zone = 256, 128
    ref_plan = mp.Plan(x, None, w, zone)
    ref_plan.prepare()
    ref_plan.run(0, 1)
    ref = {k: v.cpu().numpy() for k, v in ref_plan.outputs().items()}
    for P in (2, 3):
        plans = [mp.Plan(x, None, w, zone) for _ in range(P)]
        for s, pl in enumerate(plans):
            pl.prepare_shard(s, P)
        cks = [pl.coarse_keys() for pl in plans]
        assert all(ck is not None for ck in cks), "coarse phase expected at 1.3e9 cells"
        for j in range(2):
            m = cks[0][j].clone()
            for ck in cks[1:]:
                m = torch.minimum(m, ck[j])
            for ck in cks:
                ck[j].copy_(m)
        for s, pl in enumerate(plans):
            pl.prepare_finish()
            pl.run(s, P)
        rk0, ck0 = plans[0].keys()
        for pl in plans[1:]:
            rk, ck = pl.keys()
            rk0.copy_(torch.minimum(rk0, rk))
            ck0.copy_(torch.minimum(ck0, ck))
        got = {k: v.cpu().numpy() for k, v in plans[0].outputs().items()}
        for k in ref:
            assert np.array_equal(got[k], ref[k]), (P, k)
        for pl in plans:
            pl.close()
    ref_plan.close()
