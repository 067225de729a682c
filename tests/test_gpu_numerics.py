"""Numerically hostile inputs through the GPU join, against the oracle's
brute force (direct per-window z-normalisation):

* a random walk riding on a 1e8 offset (the centred recurrence must not lose
  the signal to the offset; the reference's raw-QT form would),
* the same series scaled by 1e-6 and by 1e+30 (z-normalisation is scale-free,
  so the profile must match the unscaled one; the fp32 paths in the kernels
  must not under- or overflow into skipped cells), and by 1e-30, where every
  window falls under the flat threshold (sd <= 1e-10 max(1, |mean|), an
  absolute floor for small data: DESIGN.md §3) and the profile is all zeros,
* a strictly periodic signal (every window has exact repeats: ties everywhere,
  the smallest index must win, MP exactly 0),
* an AB join of a series with its negation (every correlation <= 0: the filter
  must still find the least-negative cells, no key may stay empty).
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


def _walk(n, seed):
    return np.cumsum(np.random.default_rng(seed).standard_normal(n))


def _check(mp, oracle_lib, x, w, ez=0.5, y=None):
    got = mp.stomp(x, y, w, ez)
    ref = oracle_lib.brute_force_mp(x, y, w, ez)
    ok, rel = close(got.values, ref[0])
    assert ok, f"MP mismatch (max rel {rel:.3e})"
    rows = np.arange(got.values.size)
    assert not index_mismatches(got.index, ref[1], rows, x, x if y is None else y, w)
    if y is None:
        assert not index_mismatches(got.left_index, ref[2], rows, x, x, w)
        assert not index_mismatches(got.right_index, ref[3], rows, x, x, w)
    return got


def test_large_offset(mp, oracle_lib):
    x = _walk(6000, 1) + 1e8
    _check(mp, oracle_lib, x, 100)


@pytest.mark.parametrize("scale", [1e-6, 1e30])
def test_extreme_scales_match_unscaled(mp, oracle_lib, scale):
    x = _walk(5000, 2)
    base = mp.stomp(x, None, 64, 0.5)
    got = _check(mp, oracle_lib, x * scale, 64)
    ok, rel = close(got.values, base.values, rel=1e-9, abs_=1e-9)
    assert ok, f"scaled profile differs from the unscaled one (max rel {rel:.3e})"


def test_tiny_scale_is_flat(mp, oracle_lib):
    x = _walk(3000, 2) * 1e-30
    got = _check(mp, oracle_lib, x, 64)
    assert np.all(got.values == 0.0)


def test_periodic_exact_repeats(mp, oracle_lib):
    period, w = 50, 40
    one = np.sin(np.linspace(0, 2 * np.pi, period, endpoint=False)) + 0.3 * np.cos(
        np.linspace(0, 6 * np.pi, period, endpoint=False))
    x = np.tile(one, 120)
    got = _check(mp, oracle_lib, x, w)
    assert np.all(got.values[: got.values.size - period] < 1e-6)


def test_ab_anticorrelated(mp, oracle_lib):
    x = _walk(4000, 3)
    y = -x[:3000] + 1e-3 * np.random.default_rng(4).standard_normal(3000)
    got = _check(mp, oracle_lib, x, 50, y=y)
    assert np.all(got.index >= 0) and np.all(np.isfinite(got.values))


@pytest.mark.parametrize("scale,offset", [(1.0, 1e8), (1e30, 0.0), (1e-6, 0.0)])
def test_masked_anytime_on_hostile_scales(mp, scale, offset):
    """The masked band join (exact anytime SCRIMP on a dense diagonal set) marks
    the diagonals outside the set with a negative NaN covariance; neither a
    huge offset nor extreme scales may turn that into a candidate or hide one.
    Reference: direct z-normalised distances over the chosen diagonals in numpy
    (the oracle's SCRIMP uses the raw-QT recurrence, which loses the signal to a
    1e8 offset itself)."""
    n, w, ez, seed = 4000, 64, 0.5, 17
    x = _walk(n, 23) * scale + offset
    L = n - w + 1
    zone = mp.zone_size(w, ez)
    s_size = (L - zone - 1) // 3
    r = mp.scrimp(x, w, ez, s_size=s_size, seed=seed)
    diags, _ = mp.scrimp_diagonals(n, w, zone, s_size, seed)
    W = np.lib.stride_tricks.sliding_window_view(x, w)
    Z = W - W.mean(axis=1, keepdims=True)
    Z = Z / np.sqrt((Z * Z).sum(axis=1, keepdims=True) / w)  # unit population variance
    ref = np.full(L, np.inf)
    for k in diags:
        k = int(k)
        d = np.sqrt(np.maximum(((Z[:L - k] - Z[k:]) ** 2).sum(axis=1), 0.0))
        ref[:L - k] = np.minimum(ref[:L - k], d)
        ref[k:] = np.minimum(ref[k:], d)
    ok, rel = close(r.values, ref)
    assert ok, f"masked anytime at scale {scale:g} offset {offset:g}: max rel {rel:.3e}"
    fin = r.index >= 0
    assert fin.all() and np.isin(np.abs(r.index - np.arange(L)), diags).all()
    # the reported neighbour attains the reported value
    dd = np.sqrt(((Z - Z[r.index]) ** 2).sum(axis=1))
    assert close(r.values, dd)[0]
