"""The CPU oracle against the reference's pinned answers (no GPU needed).

Pins: SPEC.md known-answer examples (tests/golden/spec_kat.json), an
independent numpy brute force (tests/golden/brute_*.npz), the reference's own
compiled TimeSeries validation (oracle/_ref), and the SPEC properties
(oracle equivalence, worker determinism, zone law, profile-size law,
anytime monotonicity, merge_min identities).
"""
import json
import os

import numpy as np
import pytest

from tests.parity import index_mismatches

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def kat():
    with open(os.path.join(GOLDEN, "spec_kat.json")) as f:
        return json.load(f)


def test_rolling_stats_kat(oracle_lib, kat):
    for case in kat["rolling_mean_std"]:
        mu, sd = oracle_lib.rolling_mean_std(case["ts"], case["w"])
        assert np.allclose(mu, case["means"], atol=0) and np.allclose(sd, case["stds"], atol=0)


def test_rolling_stats_vs_direct(oracle_lib):
    """1024-sample normal draw, w = 64, within 1e-10 of direct."""
    x = np.random.default_rng(0).standard_normal(1024)
    mu, sd = oracle_lib.rolling_mean_std(x, 64)
    win = np.lib.stride_tricks.sliding_window_view(x, 64)
    assert np.max(np.abs(mu - win.mean(1))) < 1e-10
    assert np.max(np.abs(sd - win.std(1))) < 1e-10
    # reversal property (SPEC.md "Invariants"): stats of reversed series reversed
    mu_r, sd_r = oracle_lib.rolling_mean_std(x[::-1].copy(), 64)
    assert np.allclose(mu_r[::-1], mu, atol=1e-12) and np.allclose(sd_r[::-1], sd, atol=1e-12)


def test_flat_threshold(oracle_lib):
    assert oracle_lib.is_flat_std(0.0, 5.0)
    assert oracle_lib.is_flat_std(1e-16 * 1e6, 1e6)
    assert not oracle_lib.is_flat_std(1e-3, 1e3)


def test_sliding_dot_kat(oracle_lib, kat):
    for case in kat["sliding_dot_product"]:
        assert np.array_equal(oracle_lib.sliding_dot_direct(case["query"], case["ts"]), case["out"])
    assert np.all(oracle_lib.sliding_dot_direct(np.zeros(8), np.arange(20.0)) == 0)
    g = np.random.default_rng(1)
    q, t = g.standard_normal(32), g.standard_normal(512)
    ref = np.correlate(t, q, mode="valid")
    assert np.max(np.abs(oracle_lib.sliding_dot_direct(q, t) - ref)) < 1e-9


def test_zone_size_kat(oracle_lib, kat):
    for case in kat["zone_size"]:
        assert oracle_lib.zone_size(case["w"], case["fraction"]) == case["zone"]
    with pytest.raises(ValueError):
        oracle_lib.zone_size(50, -0.1)


def test_exclusion_zone_kat(oracle_lib, kat):
    c = kat["exclusion_zone"][0]
    dp = oracle_lib.apply_exclusion_zone(np.ones(c["length"]), c["center"], c["zone"])
    assert np.isfinite(dp).sum() == c["finite_remaining"]
    lo, hi = c["inf_range"]
    assert np.all(np.isinf(dp[lo:hi + 1])) and np.isfinite(dp[lo - 1]) and np.isfinite(dp[hi + 1])
    assert np.all(np.isinf(oracle_lib.apply_exclusion_zone(np.ones(10), 3, 20)))
    one = oracle_lib.apply_exclusion_zone(np.ones(10), 3, 0)
    assert np.isinf(one[3]) and np.isfinite(one).sum() == 9


def test_znorm_dist_convention(oracle_lib):
    assert oracle_lib.znorm_dist_from_qt(5.0, 16, 1.0, 0.0, 2.0, 0.0) == 0.0
    assert oracle_lib.znorm_dist_from_qt(5.0, 16, 1.0, 0.0, 2.0, 1.0) == 4.0  # sqrt(w)
    # identical windows -> 0 (clamped), anti-correlated -> 2 sqrt(w)
    w, mu, sd = 16, 0.0, 1.0
    assert oracle_lib.znorm_dist_from_qt(w * sd * sd, w, mu, sd, mu, sd) == 0.0
    assert abs(oracle_lib.znorm_dist_from_qt(-w * sd * sd, w, mu, sd, mu, sd) - 2 * np.sqrt(w)) < 1e-12


@pytest.mark.parametrize("name", ["brute_self_0", "brute_self_1", "brute_self_2", "brute_self_3",
                                  "brute_self_flat_planted", "brute_ab_0"])
def test_oracle_vs_golden_brute(oracle_lib, name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    a, w, ez = g["a"], int(g["w"]), float(g["ez"])
    b = g["b"] if "b" in g.files else None
    for fn in (oracle_lib.brute_force_mp, oracle_lib.stomp):
        mp, pi, le, ri = fn(a, b, w, ez)
        fin = np.isfinite(g["mp"])
        assert np.array_equal(np.isfinite(mp), fin)
        assert np.max(np.abs(mp[fin] - g["mp"][fin])) < 1e-8, fn.__name__
        # indices: identical except exact ties of the golden distance
        bad = (pi != g["pi"]) & (np.abs(mp - g["mp"]) > 1e-8)
        assert not bad.any(), fn.__name__
        if b is None:  # left / right: identical except near-ties of the exact distances
            rows = np.arange(le.size)
            assert not index_mismatches(le, g["left"], rows, a, a, w), fn.__name__
            assert not index_mismatches(ri, g["right"], rows, a, a, w), fn.__name__


def test_brute_planted_repeat_and_ab_identity(oracle_lib):
    """SPEC.md:191-192."""
    t = np.arange(200)
    x = np.sin(2 * np.pi * t / 100.0)
    mp, pi, _, _ = oracle_lib.brute_force_mp(x, None, 50, 0.5)
    i = int(np.argmin(mp))
    assert mp[i] < 1e-6 and abs(pi[i] - i) == 100
    y = np.random.default_rng(2).standard_normal(300)
    mp, pi, _, _ = oracle_lib.brute_force_mp(y, y.copy(), 20, 0.5)
    assert np.all(mp < 1e-6) and np.array_equal(pi, np.arange(mp.size))


def test_stomp_constant_series(oracle_lib, kat):
    c = kat["stomp_constant"]
    mp, pi, le, ri = oracle_lib.stomp(np.full(c["n"], 2.5), None, c["w"], c["ez"])
    assert np.all(mp == 0.0)
    zone = oracle_lib.zone_size(c["w"], c["ez"])
    L = c["n"] - c["w"] + 1
    for i in range(L):  # nearest admissible neighbour: smallest index on ties
        exp = 0 if i - zone - 1 >= 0 else i + zone + 1
        assert pi[i] == exp


def test_profile_size_and_zone_law(oracle_lib, kat):
    g = np.random.default_rng(3)
    for case in kat["profile_size"]:
        x = np.cumsum(g.standard_normal(case["n"]))
        assert oracle_lib.zone_size(case["w"], case["ez"]) == case["zone"]
        if case["n"] <= 1000:
            mp, pi, le, ri = oracle_lib.stomp(x, None, case["w"], case["ez"])
            assert mp.size == case["size"]
            fin = np.isfinite(mp)
            assert np.all(np.abs(pi[fin] - np.arange(mp.size)[fin]) > case["zone"])
            assert np.all(le[le >= 0] < np.arange(mp.size)[le >= 0])
            assert np.all(ri[ri >= 0] > np.arange(mp.size)[ri >= 0])


def test_oracle_equivalence_sweep(oracle_lib):
    """stomp and scrimp equal brute within 1e-8 on 50 seeded inputs."""
    g = np.random.default_rng(1904)
    for t in range(50):
        n = int(g.integers(128, 1025))
        w = int(g.integers(8, n // 4 + 1))
        ez = (0.0, 0.25, 0.5)[t % 3]
        x = np.cumsum(g.standard_normal(n))
        bf = oracle_lib.brute_force_mp(x, None, w, ez)
        st = oracle_lib.stomp(x, None, w, ez, n_workers=2)
        sc = oracle_lib.scrimp(x, w, ez, 0, t)
        fin = np.isfinite(bf[0])
        for got in (st, sc):
            assert np.array_equal(np.isfinite(got[0]), fin)
            if fin.any():
                assert np.max(np.abs(got[0][fin] - bf[0][fin])) < 1e-8
            assert np.array_equal(got[1], bf[1])


def test_worker_determinism(oracle_lib):
    """bit-identical for n_workers in {1, 2, 4, 8}."""
    x = np.cumsum(np.random.default_rng(4).standard_normal(12000))
    outs = [oracle_lib.stomp(x, None, 32, 0.5, n_workers=k) for k in (1, 2, 4, 8)]
    for o in outs[1:]:
        for u, v in zip(o, outs[0]):
            assert np.array_equal(u, v)


def test_scrimp_anytime_monotone(oracle_lib):
    x = np.cumsum(np.random.default_rng(5).standard_normal(600))
    full = oracle_lib.scrimp(x, 30, 0.5, 0, 11)
    part = oracle_lib.scrimp(x, 30, 0.5, 50, 11)
    more = oracle_lib.scrimp(x, 30, 0.5, 200, 11)
    assert part[4] < more[4] < full[4] == 1.0
    assert np.all(part[0] >= more[0]) and np.all(more[0] >= full[0])
    assert np.all(part[2] == -1) and np.all(part[3] == -1)  # left/right only at full coverage


def test_merge_min_identities(oracle_lib):
    acc = np.full(5, np.inf)
    idx = np.full(5, -1, np.int64)
    oracle_lib.merge_min(acc, idx, np.full(5, np.inf), 3)
    assert np.all(np.isinf(acc)) and np.all(idx == -1)
    dp = np.array([1.0, 2.0, np.inf, 0.5, 3.0])
    oracle_lib.merge_min(acc, idx, dp, 7)
    assert np.array_equal(acc, dp) and np.array_equal(idx, [7, 7, -1, 7, 7])
    oracle_lib.merge_min(acc, idx, dp, 9)  # ties keep the incumbent
    assert np.array_equal(idx, [7, 7, -1, 7, 7])


def test_reference_timeseries_validation(oracle_lib):
    """The reference's own compiled TimeSeries ctor (types.cpp:7-18)."""
    try:
        rc, msg = oracle_lib.ref_timeseries_validate([1.0, 2.0, 3.0])
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built (reference tree absent)")
    assert rc == 2 and "too short" in msg
    rc, msg = oracle_lib.ref_timeseries_validate([1.0, 2.0, np.inf, 4.0])
    assert rc == 2 and "not finite" in msg
    assert oracle_lib.ref_timeseries_validate([1.0, 2.0, 3.0, 4.0])[0] == 0
