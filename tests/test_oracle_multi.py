"""CPU oracle for the multivariate joins (SiMPle, mSTOMP; profile.hpp:91-100)
pinned against independent numpy brute force and the SPEC.md examples
(SPEC.md:100-106, 225-243, 262, 643-644). No GPU needed."""
import numpy as np
import pytest

from tests.parity import exact_dist, mstomp_cell, mstomp_order, raw_exact


def _walk(g, d, n):
    return np.cumsum(g.standard_normal((d, n)), axis=1)


def numpy_simple(a, b, m, zone):
    La = a.shape[1] - m + 1
    Lb = b.shape[1] - m + 1
    mp = np.full(La, np.inf)
    pi = np.full(La, -1)
    for j in range(La):
        for i in range(Lb):
            if b is a and abs(i - j) <= zone:
                continue
            v = raw_exact(a, j, b, i, m)
            if v < mp[j]:
                mp[j], pi[j] = v, i
    return mp, pi


def numpy_mstomp(x, m, zone, must=(), exc=()):
    order, nm = mstomp_order(x.shape[0], must, exc)
    D = len(order)
    L = x.shape[1] - m + 1
    v = np.full((x.shape[0], L), np.inf)
    p = np.full((x.shape[0], L), -1)
    do = np.full((x.shape[0], L), -1)
    for j in range(L):
        for i in range(L):
            if abs(i - j) <= zone:
                continue
            sel, pk, _ = mstomp_cell(x, i, j, m, order, nm)
            for k in range(D):
                if pk[k] < v[k, j]:
                    v[k, j], p[k, j], do[k, j] = pk[k], i, sel[k]
    for k in range(D, x.shape[0]):
        v[k], p[k] = v[D - 1], p[D - 1]
    return v, p, do


def test_raw_distance_profile_kats(oracle_lib):
    g = np.random.default_rng(3)
    x = _walk(g, 2, 128)
    w = 8
    # query = window of the series -> 0 there
    dp = oracle_lib.raw_distance_profile(x[:, 30:30 + w], x)
    assert dp[30] == 0.0
    # constant shift c on every dim -> sqrt(d w c^2)
    c = 0.75
    dp = oracle_lib.raw_distance_profile(x[:, 30:30 + w] + c, x)
    assert abs(dp[30] - np.sqrt(2 * w * c * c)) < 1e-12
    # random 2-dim n=128 w=8 equals the direct per-window computation
    q = g.standard_normal((2, w))
    dp = oracle_lib.raw_distance_profile(q, x)
    direct = np.array([np.sqrt(np.sum((x[:, i:i + w] - q) ** 2)) for i in range(128 - w + 1)])
    assert np.max(np.abs(dp - direct)) < 1e-9


def test_raw_terms():
    import oracle
    assert oracle.raw_sq_term(1.0, 1.0, 1.5) == 0.0          # clamped at 0
    assert oracle.raw_sq_term(2.0, 3.0, 1.0) == 3.0
    assert oracle.raw_distance_from_terms(1e-13, 1.0) == 0.0  # residue snapped
    assert oracle.raw_distance_from_terms(4.0, 1.0) == 2.0


@pytest.mark.parametrize("d,n,w", [(1, 120, 8), (2, 150, 10), (3, 97, 6)])
def test_simple_vs_numpy_brute(oracle_lib, d, n, w):
    g = np.random.default_rng(d * 100 + n)
    a = _walk(g, d, n)
    zone = oracle_lib.zone_size(w, 0.5)
    rm, rp = numpy_simple(a, a, w, zone)
    mp, pi, le, ri = oracle_lib.simple_join(a, None, w, 0.5, n_workers=2)
    assert np.max(np.abs(mp - rm) / np.maximum(rm, 1e-3)) < 1e-9
    bm, bp = oracle_lib.simple_brute(a, None, w, 0.5)
    assert np.max(np.abs(bm - rm)) < 1e-12 and np.array_equal(bp, rp)
    assert np.array_equal(pi, rp)
    # left / right: strict sides, MP = min(left, right)
    L = n - w + 1
    for i in range(L):
        if le[i] >= 0:
            assert le[i] < i
        if ri[i] >= 0:
            assert ri[i] > i


def test_simple_ab_self_identity(oracle_lib):
    """mts_b = mts_a as an AB-join: values 0, index[i] = i."""
    g = np.random.default_rng(11)
    a = g.standard_normal((3, 300))
    mp, pi, _, _ = oracle_lib.simple_join(a, a, 16, 0.5)
    assert np.all(mp == 0.0) and np.array_equal(pi, np.arange(mp.size))


def test_simple_ab_vs_numpy(oracle_lib):
    g = np.random.default_rng(12)
    a, b = _walk(g, 2, 140), _walk(g, 2, 90)
    rm, rp = numpy_simple(a, b, 12, 0)
    mp, pi, le, ri = oracle_lib.simple_join(a, b, 12, 0.5)
    assert le is None and ri is None
    assert np.max(np.abs(mp - rm) / np.maximum(rm, 1e-3)) < 1e-9
    assert np.array_equal(pi, rp)


def test_simple_matches_stomp_on_normalised_windows(oracle_lib):
    """d = 1 data whose every window has mean 0 and sigma 1 -> SiMPle values
    equal the z-normalised stomp values."""
    w, n = 64, 1200
    t = np.arange(n)
    g = np.random.default_rng(5)
    x = np.zeros(n)
    for p in (2, 4, 8):  # integer periods per window: every window has mean 0
        x += g.uniform(0.5, 1.5) * np.sin(2 * np.pi * p * t / w + g.uniform(0, 6.28))
    # every window has the same energy; scale to sigma = 1
    x /= np.sqrt(np.mean(x[:w] ** 2))
    sm, _, _, _ = oracle_lib.simple_join(x, None, w, 0.5)
    st, _, _, _ = oracle_lib.stomp(x, None, w, 0.5)
    assert np.max(np.abs(sm - st)) < 1e-6


def test_simple_worker_determinism(oracle_lib):
    g = np.random.default_rng(9)
    a = _walk(g, 2, 9000)
    r1 = oracle_lib.simple_join(a, None, 32, 0.5, n_workers=1, row_begin=0, row_end=0)
    r3 = oracle_lib.simple_join(a, None, 32, 0.5, n_workers=3)
    for u, v in zip(r1, r3):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("must,exc", [((), ()), ((2,), ()), ((), (1,)), ((3, 0), (2,))])
def test_mstomp_vs_numpy_brute(oracle_lib, must, exc):
    g = np.random.default_rng(21 + len(must) + 3 * len(exc))
    x = _walk(g, 4, 90)
    w = 8
    zone = oracle_lib.zone_size(w, 0.5)
    rv, rp, rd = numpy_mstomp(x, w, zone, must, exc)
    v, p, do = oracle_lib.mstomp(x, w, 0.5, must, exc, n_workers=2)
    D = 4 - len(exc)
    assert np.max(np.abs(v - rv) / np.maximum(rv, 1e-3)) < 1e-9
    assert np.array_equal(p, rp)
    assert np.array_equal(do[:D], rd[:D]) and np.all(do[D:] == -1)


def test_mstomp_properties(oracle_lib):
    g = np.random.default_rng(31)
    x = _walk(g, 3, 400)
    w = 16
    v, p, do = oracle_lib.mstomp(x, w, 0.5)
    # row monotonicity
    assert np.all(v[:-1] <= v[1:] + 1e-12)
    # d = 1 reduction equals stomp within 1e-8
    v1, p1, d1 = oracle_lib.mstomp(x[:1], w, 0.5)
    st, sp, _, _ = oracle_lib.stomp(x[0], None, w, 0.5)
    assert np.max(np.abs(v1[0] - st)) < 1e-8 and np.all(d1[0] == 0)
    # exclusion collapses to univariate
    v2, p2, d2 = oracle_lib.mstomp(x[:2], w, 0.5, exc_dims=(1,))
    assert np.max(np.abs(v2[0] - st)) < 1e-8 and np.array_equal(v2[1], v2[0])
    assert np.all(d2[1] == -1) and np.all(d2[0] == 0)
    # worker determinism
    va, pa, da = oracle_lib.mstomp(x, w, 0.5, n_workers=1)
    vb, pb, db = oracle_lib.mstomp(x, w, 0.5, n_workers=4)
    assert np.array_equal(va, vb) and np.array_equal(pa, pb) and np.array_equal(da, db)


def test_mstomp_parameter_errors(oracle_lib):
    x = np.random.default_rng(1).standard_normal((3, 64))
    for must, exc in (((0,), (0,)), ((), (0, 1, 2)), ((3,), ()), ((0, 0), ()), ((), (-1,))):
        with pytest.raises(ValueError):
            oracle_lib.mstomp(x, 8, 0.5, must, exc)


def planted_multivariate(seed, n=2000, m=64):
    """d = 3: dims 0 and 1 carry the same planted motif pair (two noisy copies
    of a sine burst replacing the walk), dim 2 is pure noise."""
    g = np.random.default_rng(seed)
    x = np.cumsum(g.standard_normal((3, n)), axis=1)
    x[2] = g.standard_normal(n)
    s1 = int(g.integers(0, n // 2 - 2 * m))
    s2 = int(g.integers(n // 2, n - 2 * m))
    burst = 5 * np.sin(2 * np.pi * g.uniform(1, 8) * np.arange(m) / m)
    for d in (0, 1):
        for s in (s1, s2):
            x[d, s:s + m] = x[d, s] + burst + g.normal(0, 0.1, m)
    return x, s1, s2


def test_mstomp_planted_motif(oracle_lib):
    hits = 0
    for seed in range(6):
        x, s1, s2 = planted_multivariate(seed, n=900, m=48)
        v, p, do = oracle_lib.mstomp(x, 48, 0.5, n_workers=4)
        c = int(np.argmin(v[1]))
        pair = {c, int(p[1, c])}
        near = all(min(abs(q - s1), abs(q - s2)) <= 2 for q in pair)
        dims = {int(do[0, c]), int(do[1, c])}
        hits += near and dims == {0, 1}
    assert hits >= 5
