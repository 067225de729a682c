"""Anytime SCRIMP (profile.hpp:85-89) on the GPU: a seeded
subset of 256-diagonal bands, checked against the oracle's SCRIMP loop over
exactly those diagonals, plus the anytime contract (coverage, monotonicity,
left/right absent below full coverage, full coverage == the exact join)."""
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


def _check_subset(mp, oracle_lib, x, w, ez, s_size, seed):
    r = mp.scrimp(x, w, ez, s_size=s_size, seed=seed)
    zone = mp.zone_size(w, ez)
    L = x.size - w + 1
    bands, cov = mp.scrimp_bands(x.size, w, zone, s_size, seed)
    assert r.coverage == cov < 1.0 and not r.has_left_right()
    diags = mp.band_diagonals(bands, L, zone)
    ref_mp, ref_pi = oracle_lib.scrimp_diagonals(x, w, diags)
    ok, rel = close(r.values, ref_mp)
    assert ok, f"anytime MP mismatch (max rel {rel:.3e})"
    assert not index_mismatches(r.index, ref_pi, np.arange(L), x, x, w)
    return r


def test_anytime_matches_oracle_subset(mp, oracle_lib):
    x = np.cumsum(np.random.default_rng(31).standard_normal(30000))
    w, ez = 64, 0.5
    nd = x.size - w + 1 - mp.zone_size(w, ez) - 1
    for frac, seed in ((0.05, 1), (0.3, 2)):
        _check_subset(mp, oracle_lib, x, w, ez, int(nd * frac), seed)


def test_anytime_with_flat_runs(mp, oracle_lib):
    g = np.random.default_rng(32)
    x = np.cumsum(g.standard_normal(12000))
    x[2000:2600] = x[2000]
    x[7000:7300] = 1.5
    nd = x.size - 50 + 1 - mp.zone_size(50, 0.25) - 1
    _check_subset(mp, oracle_lib, x, 50, 0.25, nd // 4, 5)
    # more chosen bands than lanes (the finalize splits the band search over the warp)
    y = np.cumsum(g.standard_normal(40000))
    y[5000:5400] = y[5000]
    y[21000:21150] = -3.0
    y[33000:33100] = y[33000]
    nd = y.size - 32 + 1 - mp.zone_size(32, 0.5) - 1
    _check_subset(mp, oracle_lib, y, 32, 0.5, nd // 2, 6)


def test_anytime_monotone_and_full(mp):
    x = np.cumsum(np.random.default_rng(33).standard_normal(20000))
    w, ez = 100, 0.5
    nd = x.size - w + 1 - mp.zone_size(w, ez) - 1
    r1 = mp.scrimp(x, w, ez, s_size=nd // 20, seed=9)
    r2 = mp.scrimp(x, w, ez, s_size=nd // 4, seed=9)
    full = mp.scrimp(x, w, ez, seed=9)
    st = mp.stomp(x, None, w, ez)
    assert r1.coverage < r2.coverage < full.coverage == 1.0
    assert np.all(r2.values <= r1.values) and np.all(full.values <= r2.values)
    assert np.array_equal(full.values, st.values) and np.array_equal(full.index, st.index)
    assert np.array_equal(full.left_index, st.left_index) and full.has_left_right()
