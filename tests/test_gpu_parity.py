"""GPU parity: the CUDA join (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): MP 1e-6 relative (1e-6 absolute floor
near 0), +inf/-1 exact, PI equal except at near-ties (tests/parity.py).
"""
import numpy as np
import pytest

from tests.parity import close, index_mismatches

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_12626_b200 as mp
    mp.lib()
    return mp


def _check_self(mp, oracle, x, w, ez, ref=None, label=""):
    got = mp.stomp(x, None, w, ez)
    if ref is None:
        ref = oracle.brute_force_mp(x, None, w, ez)
    ok, rel = close(got.values, ref[0])
    assert ok, f"{label} MP mismatch (max rel {rel:.3e})"
    L = x.size - w + 1
    rows = np.arange(L)
    for name, g, r in (("PI", got.index, ref[1]), ("left", got.left_index, ref[2]),
                       ("right", got.right_index, ref[3])):
        bad = index_mismatches(g, r, rows, x, x, w)
        assert not bad, f"{label} {name} mismatches: {bad[:5]}"
    return got


def test_random_sweep_vs_brute(mp, oracle_lib):
    """SPEC.md:256 property: 50 seeded inputs, n in [128,1024], w in [8,n/4], ez in {0,1/4,1/2}."""
    g = np.random.default_rng(1904)
    for t in range(50):
        n = int(g.integers(128, 1025))
        w = int(g.integers(8, n // 4 + 1))
        ez = (0.0, 0.25, 0.5)[t % 3]
        x = np.cumsum(g.standard_normal(n))
        _check_self(mp, oracle_lib, x, w, ez, label=f"case {t} n={n} w={w} ez={ez}")


def test_c1_vs_oracle_stomp_and_brute(mp, oracle_lib):
    from paper_1904_12626_b200 import datasets
    c = datasets.c1()
    ref = oracle_lib.stomp(c.a, None, c.window, c.ez, n_workers=oracle_lib.default_threads())
    _check_self(mp, oracle_lib, c.a, c.window, c.ez, ref=ref, label="C1/stomp")
    bf = oracle_lib.brute_force_mp(c.a, None, c.window, c.ez)
    _check_self(mp, oracle_lib, c.a, c.window, c.ez, ref=bf, label="C1/brute")


def test_edge_cases(mp, oracle_lib):
    g = np.random.default_rng(7)
    # L = 1 (n == w): nothing admissible
    x = g.standard_normal(16)
    r = mp.stomp(x, None, 16, 0.5)
    assert r.values.size == 1 and np.isinf(r.values[0]) and r.index[0] == -1
    # zone >= L - 1: all +inf / -1
    x = np.cumsum(g.standard_normal(40))
    r = mp.stomp(x, None, 20, 1.0)
    assert np.all(np.isinf(r.values)) and np.all(r.index == -1)
    assert np.all(r.left_index == -1) and np.all(r.right_index == -1)
    # minimum window 4
    x = np.cumsum(g.standard_normal(300))
    _check_self(mp, oracle_lib, x, 4, 0.5, label="w=4")
    # constant series -> all 0, index = nearest admissible
    c = np.full(64, 3.25)
    r = mp.stomp(c, None, 8, 0.5)
    ref = oracle_lib.stomp(c, None, 8, 0.5)
    assert np.all(r.values == 0.0)
    assert np.array_equal(r.index, ref[1])
    assert np.array_equal(r.left_index, ref[2]) and np.array_equal(r.right_index, ref[3])
    # negative best correlations: a pure sine at half-period spacing
    t = np.arange(400)
    s = np.sin(2 * np.pi * t / 37.0) + 1e-3 * g.standard_normal(400)
    _check_self(mp, oracle_lib, s, 30, 0.5, label="sine")


def test_flat_windows_convention(mp, oracle_lib):
    g = np.random.default_rng(11)
    x = np.cumsum(g.standard_normal(3000))
    x[500:900] = x[500]       # flat run: windows inside are flat
    x[2000:2150] = -7.5       # second flat run
    for w, ez in ((64, 0.5), (100, 0.25), (32, 0.0)):
        _check_self(mp, oracle_lib, x, w, ez, label=f"flat w={w} ez={ez}")


def test_ab_join_both_directions(mp, oracle_lib):
    g = np.random.default_rng(5)
    a = np.cumsum(g.standard_normal(20000))
    b = np.cumsum(g.standard_normal(5000))
    w = 128
    pa, pb = mp.stomp_ab(a, b, w)
    ra = oracle_lib.stomp(a, b, w)
    rb = oracle_lib.stomp(b, a, w)
    ok, rel = close(pa.values, ra[0])
    assert ok, f"A-profile rel {rel:.3e}"
    ok, rel = close(pb.values, rb[0])
    assert ok, f"B-profile rel {rel:.3e}"
    assert not index_mismatches(pa.index, ra[1], np.arange(pa.size()), a, b, w)
    assert not index_mismatches(pb.index, rb[1], np.arange(pb.size()), b, a, w)


def test_ab_join_with_itself_is_identity(mp):
    """AB-join of a series with itself -> 0 and index[i] = i."""
    x = np.random.default_rng(3).standard_normal(2000)
    r = mp.stomp(x, x.copy(), 50, 0.5)
    assert np.all(r.values == 0.0)  # exact: distances recomputed without FMA contraction
    assert np.array_equal(r.index, np.arange(r.size()))


def test_virtual_shards_bit_identical(mp):
    """Sharded execution (1 GPU, P shards) equals P = 1 bit for bit."""
    import torch
    x = np.cumsum(np.random.default_rng(9).standard_normal(40000))
    d = torch.from_numpy(x).cuda()
    plan = mp.Plan(d, None, 128, 64)
    outs = []
    for P in (1, 3, 8):
        plan.prepare()
        for s in range(P):
            plan.run(s, P)
        o = plan.outputs()
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in o.items()})
    for o in outs[1:]:
        for k in o:
            assert np.array_equal(o[k], outs[0][k], equal_nan=True), k
    # and the keys of separate shards min-merge to the same keys
    assert sum(plan.cells(s, 8) for s in range(8)) == plan.cells(0, 1) == mp.join_cells(40000, 0, 128, 64)
    plan.close()


def test_multi_context_join_matches_single(mp):
    """mpgpu_join over several shard contexts (fused peer-key merge path; on one
    GPU the 'peers' are virtual shards on the same device)."""
    g = np.random.default_rng(21)
    x = np.cumsum(g.standard_normal(30000))
    r1 = mp.join(x, None, 100, 50)
    for devs in ([0, 0], [0, 0, 0]):
        r2 = mp.join(x, None, 100, 50, devices=devs)
        for k in r1:
            assert np.array_equal(r1[k], r2[k]), (devs, k)
    y = np.cumsum(g.standard_normal(7000))
    a1 = mp.join(x, y, 64, 0)
    a2 = mp.join(x, y, 64, 0, devices=[0, 0])
    for k in a1:
        assert np.array_equal(a1[k], a2[k]), k


def test_ab_join_edge_shapes(mp, oracle_lib):
    """AB-joins with a one-window side, a side shorter than a band, and equal lengths."""
    g = np.random.default_rng(61)
    cases = [(300, 40, 40), (40, 300, 40), (5000, 120, 64), (120, 5000, 64), (777, 777, 50), (64, 64, 64)]
    for na, nb, w in cases:
        a = np.cumsum(g.standard_normal(na))
        b = np.cumsum(g.standard_normal(nb))
        pa, pb = mp.stomp_ab(a, b, w)
        ra = oracle_lib.brute_force_mp(a, b, w)
        rb = oracle_lib.brute_force_mp(b, a, w)
        assert close(pa.values, ra[0])[0] and close(pb.values, rb[0])[0], (na, nb, w)
        assert not index_mismatches(pa.index, ra[1], np.arange(pa.size()), a, b, w), (na, nb, w)
        assert not index_mismatches(pb.index, rb[1], np.arange(pb.size()), b, a, w), (na, nb, w)


def test_scrimp_ab_unsupported_on_gpu_api(mp):
    x = np.cumsum(np.random.default_rng(62).standard_normal(500))
    with pytest.raises(mp.UnsupportedError):
        mp.scrimp(x, 20, 0.5, ts_b=x)
    import ctypes
    args = mp._JoinArgs()
    a = np.ascontiguousarray(x)
    args.a = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    args.n_a = a.size
    args.b = args.a
    args.n_b = a.size
    args.window = 20
    cov = ctypes.c_double()
    assert mp.lib().mpgpu_scrimp(ctypes.byref(args), 10, 0, ctypes.byref(cov)) == mp.MPGPU_EUNSUPPORTED
