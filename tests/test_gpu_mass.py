"""MASS distance-profile batch (mass_distance_profile, distance.hpp:26-33) on
the GPU against the oracle, plus the SPEC.md:95-98,131-132 properties."""
import numpy as np
import pytest

from tests.parity import close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_12626_b200 as mp
    mp.lib()
    return mp


def test_mass_self_queries_vs_oracle(mp, oracle_lib):
    import torch
    g = np.random.default_rng(41)
    x = np.cumsum(g.standard_normal(20000))
    x[5000:5600] = x[5000]  # flat run
    w, zone = 128, 64
    pos = np.array([0, 17, 5100, 9999, 19872 - 1], dtype=np.int64)
    d = torch.from_numpy(x).cuda()
    out = mp.distance_profiles(d, w, positions=torch.from_numpy(pos).cuda(), zone=zone).cpu().numpy()
    for k, p in enumerate(pos):
        ref = oracle_lib.mass_distance_profile(x[p:p + w], x, int(p), zone)
        ok, rel = close(out[k], ref, rel=1e-9, abs_=1e-9)
        assert ok, f"query {p}: rel {rel:.3e}"


def test_mass_external_queries_and_properties(mp, oracle_lib):
    import torch
    g = np.random.default_rng(42)
    ts = g.standard_normal(256)
    w = 16
    q = ts[10:26].copy()
    # self-distance 0, affine invariance, brute-force equality
    prof = mp.mass_distance_profile(q, ts)
    assert prof[10] == 0.0 and np.all(prof >= 0)
    prof2 = mp.mass_distance_profile(3.0 + 2.5 * q, ts)
    assert np.max(np.abs(prof2 - prof)) < 1e-9
    ref = oracle_lib.mass_distance_profile(q, ts)
    assert np.max(np.abs(prof - ref)) < 1e-9
    # a batch of external queries, including a constant (flat) one
    qs = np.stack([g.standard_normal(w) for _ in range(6)] + [np.full(w, 2.0)])
    out = mp.distance_profiles(torch.from_numpy(ts).cuda(), w,
                               queries=torch.from_numpy(qs).cuda()).cpu().numpy()
    for k in range(qs.shape[0]):
        ok, rel = close(out[k], oracle_lib.mass_distance_profile(qs[k], ts), rel=1e-9, abs_=1e-9)
        assert ok, k
    assert np.allclose(out[-1], np.sqrt(w))  # flat query vs non-flat windows


def test_mass_row_equals_join_minimum(mp):
    """min over a self-query's profile == MP at that position (consistency with the join)."""
    import torch
    x = np.cumsum(np.random.default_rng(43).standard_normal(8000))
    w = 100
    zone = mp.zone_size(w, 0.5)
    prof = mp.stomp(x, None, w, 0.5)
    pos = np.array([5, 1234, 4000, 7800], dtype=np.int64)
    out = mp.distance_profiles(torch.from_numpy(x).cuda(), w, positions=torch.from_numpy(pos).cuda(),
                               zone=zone).cpu().numpy()
    for k, p in enumerate(pos):
        j = int(np.argmin(out[k]))
        assert abs(out[k][j] - prof.values[p]) <= 1e-9 * max(1.0, prof.values[p])
        assert j == prof.index[p]


def test_constant_memory_and_shared_memory_query_paths_agree(mp, tmp_path):
    """k_mass<true> (queries as constant-bank operands, several launches when
    they do not fit one) against k_mass<false> (queries staged in shared
    memory; MPGPU_MASS_CONST=0, read once per process, hence the child): the
    same sums in the same order, so the same bits. 70 queries of 300 samples
    take three constant-memory launches; a 7,200-sample window exceeds the
    constant buffer and runs the shared-memory form in this process too."""
    import os
    import subprocess
    import sys
    import torch
    g = np.random.default_rng(5)
    x = np.cumsum(g.standard_normal(60000))
    x[700:1400] = x[700]
    w, zone = 300, 150
    pos = np.sort(g.choice(x.size - w, size=70, replace=False)).astype(np.int64)
    pos[0] = 800  # a flat query
    np.savez(tmp_path / "in.npz", x=x, pos=pos)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    child = (f"import sys, numpy as np, torch; sys.path.insert(0, {root!r}); import paper_1904_12626_b200 as mp; "
             f"d = np.load({str(tmp_path / 'in.npz')!r}); "
             f"o = mp.distance_profiles(torch.from_numpy(d['x']).cuda(), {w}, "
             f"positions=torch.from_numpy(d['pos']).cuda(), zone={zone}); "
             f"np.save({str(tmp_path / 'shared.npy')!r}, o.cpu().numpy())")
    subprocess.run([sys.executable, "-c", child], check=True, timeout=600,
                   env=dict(os.environ, MPGPU_MASS_CONST="0"))
    out = mp.distance_profiles(torch.from_numpy(x).cuda(), w, positions=torch.from_numpy(pos).cuda(),
                               zone=zone).cpu().numpy()
    assert np.array_equal(out, np.load(tmp_path / "shared.npy"))
    # a window longer than the constant buffer
    wl = 7200
    y = np.cumsum(g.standard_normal(3 * wl))
    q = torch.from_numpy(np.array([0, wl // 2], dtype=np.int64)).cuda()
    o = mp.distance_profiles(torch.from_numpy(y).cuda(), wl, positions=q, zone=-1).cpu().numpy()
    assert o[0, 0] == 0.0 and o[1, wl // 2] == 0.0 and np.all(np.isfinite(o))
