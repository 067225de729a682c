"""GPU parity for the multivariate joins (SiMPle, mSTOMP; profile.hpp:91-100)
through the C ABI (mpgpu_simple_join / mpgpu_mstomp) against the CPU oracle.

Bar as for the univariate join: values within 1e-6 relative (1e-6 absolute
near 0), +inf / -1 exact, indexes (and mSTOMP dim_order) identical except at
near-ties of the exactly recomputed values (tests/parity.py)."""
import numpy as np
import pytest

from tests.parity import close, mstomp_mismatches, raw_index_mismatches

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_12626_b200 as mp
    mp.lib()
    return mp


def _walk(g, d, n):
    return np.cumsum(g.standard_normal((d, n)), axis=1)


def _check_simple_self(mp, oracle, a, w, ez, label):
    got = mp.simple_join(a, None, w, ez)
    ref = oracle.simple_join(a, None, w, ez, n_workers=oracle.default_threads())
    ok, rel = close(got.values, ref[0])
    assert ok, f"{label}: values (max rel {rel:.3e})"
    rows = np.arange(got.values.size)
    for name, g, r in (("index", got.index, ref[1]), ("left", got.left_index, ref[2]),
                       ("right", got.right_index, ref[3])):
        bad = raw_index_mismatches(g, r, rows, a, a, w)
        assert not bad, f"{label}: {name} {bad[:4]}"


def test_simple_self_sweep(mp, oracle_lib):
    g = np.random.default_rng(1904)
    for t in range(24):
        d = int(g.integers(1, 6))
        n = int(g.integers(64, 900))
        w = int(g.integers(4, max(5, n // 4)))
        ez = (0.0, 0.25, 0.5)[t % 3]
        _check_simple_self(mp, oracle_lib, _walk(g, d, n), w, ez, f"case {t} d={d} n={n} w={w}")


def test_simple_ab_both_directions(mp, oracle_lib):
    g = np.random.default_rng(7)
    for d, na, nb, w in ((1, 700, 300, 32), (3, 256, 513, 16), (4, 96, 96, 8)):
        a, b = _walk(g, d, na), _walk(g, d, nb)
        pa, pb = mp.simple_join(a, b, w, want_b=True)
        ra = oracle_lib.simple_join(a, b, w)
        rb = oracle_lib.simple_join(b, a, w)
        for got, ref, x, y in ((pa, ra, a, b), (pb, rb, b, a)):
            ok, rel = close(got.values, ref[0])
            assert ok, f"AB d={d}: values (max rel {rel:.3e})"
            bad = raw_index_mismatches(got.index, ref[1], np.arange(got.values.size), x, y, w)
            assert not bad, bad[:4]
        assert pa.join_kind == "ab" and pa.left_index.size == 0


def test_simple_ab_self_identity(mp):
    """mts_b = mts_a, no zone -> values 0 and index[i] = i."""
    a = np.random.default_rng(3).standard_normal((3, 2000))
    p = mp.simple_join(a, a, 40)
    assert np.all(p.values == 0.0)
    assert np.array_equal(p.index, np.arange(p.values.size))


def test_simple_planted_chroma(mp):
    """d = 12, two copies of a 40-column pattern in noise, w = 20."""
    hits = 0
    for seed in range(10):
        g = np.random.default_rng(seed)
        x = g.uniform(0, 1, (12, 1500))
        pat = g.uniform(0, 1, (12, 40))
        s1, s2 = int(g.integers(0, 600)), int(g.integers(800, 1400))
        x[:, s1:s1 + 40] = pat + g.normal(0, 0.01, pat.shape)
        x[:, s2:s2 + 40] = pat + g.normal(0, 0.01, pat.shape)
        p = mp.simple_join(x, None, 20, 0.5)
        c = int(np.argmin(p.values))
        j = int(p.index[c])
        hits += (s1 <= c <= s1 + 20 and s2 <= j <= s2 + 20) or (s2 <= c <= s2 + 20 and s1 <= j <= s1 + 20)
    assert hits >= 9


def test_simple_flat_runs_and_shift(mp, oracle_lib):
    g = np.random.default_rng(17)
    a = _walk(g, 2, 1200) + 1e4          # large offset: cancellation in the raw QT form
    a[0, 200:400] = 3.0
    a[1, 600:700] = -2.0
    _check_simple_self(mp, oracle_lib, a, 24, 0.5, "flat+offset")


def test_simple_larger(mp, oracle_lib):
    g = np.random.default_rng(23)
    _check_simple_self(mp, oracle_lib, _walk(g, 3, 12000), 64, 0.5, "d=3 n=12000")


def _check_mstomp(mp, oracle, x, w, ez=0.5, must=(), exc=(), label=""):
    got = mp.mstomp(x, w, ez, must, exc)
    ref = oracle.mstomp(x, w, ez, must, exc, n_workers=oracle.default_threads())
    bad = mstomp_mismatches((got.values, got.index, got.dim_order), ref, x, w, must, exc)
    assert not bad, f"{label}: {bad[:4]}"
    return got


def test_mstomp_sweep(mp, oracle_lib):
    g = np.random.default_rng(2019)
    for t in range(16):
        d = int(g.integers(1, 7))
        n = int(g.integers(64, 700))
        w = int(g.integers(4, max(5, n // 4)))
        ez = (0.0, 0.25, 0.5)[t % 3]
        _check_mstomp(mp, oracle_lib, _walk(g, d, n), w, ez, label=f"case {t} d={d} n={n} w={w}")


@pytest.mark.parametrize("must,exc", [((2,), ()), ((), (1,)), ((3, 0), (2,)), ((1,), (0, 4))])
def test_mstomp_must_exc(mp, oracle_lib, must, exc):
    g = np.random.default_rng(5 + len(must))
    _check_mstomp(mp, oracle_lib, _walk(g, 5, 500), 24, 0.5, must, exc, label=f"{must}/{exc}")


def test_mstomp_many_dims(mp, oracle_lib):
    """d > 8 runs the capacity-12 / 16 kernels with padding slots."""
    g = np.random.default_rng(41)
    _check_mstomp(mp, oracle_lib, _walk(g, 10, 300), 16, label="d=10")
    _check_mstomp(mp, oracle_lib, _walk(g, 14, 200), 12, exc=(3,), label="d=14")


def test_mstomp_reductions(mp, oracle_lib):
    g = np.random.default_rng(43)
    x = _walk(g, 2, 3000)
    w = 64
    st = mp.stomp(x[0], None, w, 0.5)
    one = mp.mstomp(x[:1], w, 0.5)
    assert np.max(np.abs(one.values[0] - st.values)) < 1e-8
    assert np.all(one.dim_order[0] == 0)
    ex = mp.mstomp(x, w, 0.5, exc_dims=(1,))
    assert np.max(np.abs(ex.values[0] - st.values)) < 1e-8
    assert np.array_equal(ex.values[1], ex.values[0]) and np.all(ex.dim_order[1] == -1)
    full = mp.mstomp(x, w, 0.5)
    assert np.all(full.values[0] <= full.values[1] + 1e-12)


def test_mstomp_flat_windows(mp, oracle_lib):
    g = np.random.default_rng(47)
    x = _walk(g, 3, 900)
    x[0, 100:300] = 1.5
    x[2, 500:800] = 0.0
    _check_mstomp(mp, oracle_lib, x, 32, label="flat")


def test_mstomp_planted_motif(mp):
    from tests.test_oracle_multi import planted_multivariate
    hits = 0
    for seed in range(20):
        x, s1, s2 = planted_multivariate(seed, n=3000, m=64)
        r = mp.mstomp(x, 64, 0.5)
        c = int(np.argmin(r.values[1]))
        pair = {c, int(r.index[1, c])}
        near = all(min(abs(q - s1), abs(q - s2)) <= 2 for q in pair)
        hits += near and {int(r.dim_order[0, c]), int(r.dim_order[1, c])} == {0, 1}
    assert hits >= 18


def test_mstomp_larger(mp, oracle_lib):
    g = np.random.default_rng(53)
    _check_mstomp(mp, oracle_lib, _walk(g, 3, 6000), 128, label="d=3 n=6000")


def test_multivariate_errors(mp):
    x = np.random.default_rng(1).standard_normal((3, 64))
    for must, exc in (((0,), (0,)), ((), (0, 1, 2)), ((3,), ()), ((0, 0), ()), ((), (-1,))):
        with pytest.raises(mp.ParameterError):
            mp.mstomp(x, 8, 0.5, must, exc)
    with pytest.raises(mp.ParameterError):
        mp.simple_join(x, x[:2], 8)                                # dimension mismatch
    with pytest.raises(mp.ParameterError):
        mp.simple_join(x, None, 65)                                # window > n
    with pytest.raises(mp.ParameterError):
        mp.MultiTimeSeries([x[0], x[1][:50]])                      # unequal lengths


def test_multivariate_edge_shapes(mp, oracle_lib):
    """L = 1, zone >= L - 1 (nothing admissible), w = 4, constant dims, AB with
    L_B = 1: +inf / -1 where every candidate is excluded."""
    g = np.random.default_rng(61)
    x = _walk(g, 3, 40)
    # L = 1: no partner at all
    s1 = mp.simple_join(x[:, :8], None, 8, 0.5)
    assert np.isinf(s1.values).all() and (s1.index == -1).all()
    m1 = mp.mstomp(x[:, :8], 8, 0.5)
    assert np.isinf(m1.values).all() and (m1.index == -1).all() and (m1.dim_order == -1).all()
    # zone covers everything: ez = 10 -> zone = 80 > L
    s2 = mp.simple_join(x, None, 8, 10.0)
    assert np.isinf(s2.values).all() and (s2.left_index == -1).all() and (s2.right_index == -1).all()
    m2 = mp.mstomp(x, 8, 10.0)
    assert np.isinf(m2.values).all()
    # minimum window, partially constant dims, against the oracle
    y = _walk(g, 3, 300)
    y[1] = 2.5                                   # a constant dimension
    y[0, 100:160] = -1.0
    _check_simple_self(mp, oracle_lib, y, 4, 0.5, "w=4 flats")
    _check_mstomp(mp, oracle_lib, y, 4, label="w=4 flats")
    # AB with a one-window B
    a, b = _walk(g, 2, 200), _walk(g, 2, 16)
    pa, pb = mp.simple_join(a, b, 16, want_b=True)
    ra = oracle_lib.simple_join(a, b, 16)
    assert close(pa.values, ra[0])[0] and (pa.index == 0).all()
    rb = oracle_lib.simple_join(b, a, 16)
    assert close(pb.values, rb[0])[0]


def test_mstomp_constant_series(mp, oracle_lib):
    """Every window flat in every dim: all distances 0 (flat-vs-flat), values 0."""
    x = np.ones((2, 64)) * np.array([[3.0], [-1.0]])
    r = mp.mstomp(x, 8, 0.5)
    ref = oracle_lib.mstomp(x, 8, 0.5)
    assert np.all(r.values == 0.0) and np.all(ref[0] == 0.0)
    assert np.array_equal(r.index, ref[1])           # smallest admissible partner, as the oracle


@pytest.mark.parametrize("ring", ["1", "0"])
def test_simple_many_dims(mp, oracle_lib, monkeypatch, ring):
    """d = 9-12 runs the ring kernel with one diagonal per lane (k_simple_r<1, d>);
    with the ring off (and above 12 dims) the dims-outermost tiled kernel
    (k_simple_dt) runs."""
    monkeypatch.setenv("MPGPU_SIMPLE_RING", ring)
    g = np.random.default_rng(71)
    _check_simple_self(mp, oracle_lib, _walk(g, 10, 700), 20, 0.5, "d=10")
    _check_simple_self(mp, oracle_lib, g.uniform(0, 1, (12, 900)), 16, 0.25, "d=12 uniform")
    a, b = _walk(g, 9, 500), _walk(g, 9, 300)
    pa, pb = mp.simple_join(a, b, 24, want_b=True)
    for got, ref, x, y in ((pa, oracle_lib.simple_join(a, b, 24), a, b),
                           (pb, oracle_lib.simple_join(b, a, 24), b, a)):
        assert close(got.values, ref[0])[0]
        assert not raw_index_mismatches(got.index, ref[1], np.arange(got.values.size), x, y, 24)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_simple_coarse_warm_start(mp, oracle_lib, monkeypatch, d):
    """The coarse warm start (PAA join + fine cells around its matches) forced on
    at sizes the oracle finishes quickly: self-join with flat runs, and AB both
    ways. Its cells are cells of the join, so the profile matches the oracle."""
    monkeypatch.setenv("MPGPU_SIMPLE_COARSE", "1")
    g = np.random.default_rng(300 + d)
    a = _walk(g, d, 6000)
    a[:, 2000:2300] = 1.5                              # flat run in every dim
    _check_simple_self(mp, oracle_lib, a, 64, 0.5, f"coarse d={d}")
    _check_simple_self(mp, oracle_lib, _walk(g, d, 3000), 128, 0.25, f"coarse d={d} w=128")
    x, y = _walk(g, d, 4000), _walk(g, d, 1500)
    px, py = mp.simple_join(x, y, 64, want_b=True)
    for got, ref, u, v in ((px, oracle_lib.simple_join(x, y, 64), x, y),
                           (py, oracle_lib.simple_join(y, x, 64), y, x)):
        ok, rel = close(got.values, ref[0])
        assert ok, f"coarse AB d={d}: values (max rel {rel:.3e})"
        assert not raw_index_mismatches(got.index, ref[1], np.arange(got.values.size), u, v, 64)


def test_mstomp_one_admissible_dim_on_k_join(mp, oracle_lib, monkeypatch):
    """One admissible dimension runs on the univariate join (k_join): same
    profile as the general mSTOMP kernel and the oracle, flat windows and an
    excluded dimension included (rows k >= 1 repeat row 0, dim_order -1)."""
    g = np.random.default_rng(91)
    x = _walk(g, 1, 3000)
    x[0, 1000:1200] = 2.0
    got = _check_mstomp(mp, oracle_lib, x, 64, label="d=1 on k_join")
    y = _walk(g, 3, 2000)
    y[1, 500:700] = -1.0
    got3 = _check_mstomp(mp, oracle_lib, y, 32, exc=(0, 2), label="exc -> D=1 on k_join")
    assert np.all(got3.dim_order[1:] == -1) and np.array_equal(got3.values[1], got3.values[0])
    monkeypatch.setenv("MPGPU_MSTOMP_K3", "0")
    ref = mp.mstomp(x, 64, 0.5)
    assert np.allclose(ref.values, got.values, rtol=1e-9, atol=1e-9)
    assert np.array_equal(ref.dim_order, got.dim_order)


def test_simple_above_ring_dims(mp, oracle_lib):
    """More than 12 dims: the tiled kernel by default."""
    g = np.random.default_rng(73)
    _check_simple_self(mp, oracle_lib, _walk(g, 14, 600), 16, 0.5, "d=14")

