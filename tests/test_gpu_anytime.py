"""Anytime SCRIMP (profile.hpp:85-89) on the GPU.

Exact mode (the reference's semantics, the default): exactly s_size
diagonals in SCRIMP's seeded order, checked against the oracle's own
or_scrimp with the same s_size and seed (same diagonal order), coverage ==
s_size / all diagonals. Band mode (the fast path): a seeded subset of
256-diagonal bands, checked against the oracle's SCRIMP loop over exactly
those diagonals. Plus the anytime contract (monotonicity, left/right absent
below full coverage, full coverage == the exact join) in both modes."""
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
    r = mp.scrimp(x, w, ez, s_size=s_size, seed=seed, granularity="band")
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


@pytest.mark.parametrize("gran", ["band", "diagonal"])
def test_anytime_monotone_and_full(mp, gran):
    x = np.cumsum(np.random.default_rng(33).standard_normal(20000))
    w, ez = 100, 0.5
    nd = x.size - w + 1 - mp.zone_size(w, ez) - 1
    r1 = mp.scrimp(x, w, ez, s_size=nd // 20, seed=9, granularity=gran)
    r2 = mp.scrimp(x, w, ez, s_size=nd // 4, seed=9, granularity=gran)
    full = mp.scrimp(x, w, ez, seed=9, granularity=gran)
    st = mp.stomp(x, None, w, ez)
    assert r1.coverage < r2.coverage < full.coverage == 1.0
    assert np.all(r2.values <= r1.values) and np.all(full.values <= r2.values)
    assert np.array_equal(full.values, st.values) and np.array_equal(full.index, st.index)
    assert np.array_equal(full.left_index, st.left_index) and full.has_left_right()


@pytest.mark.parametrize("n,w,ez,frac,seed", [(30000, 64, 0.5, 0.1, 1), (12000, 50, 0.25, 0.37, 5),
                                             (5000, 32, 0.5, 1e-4, 3), (40000, 128, 0.5, 0.02, 11),
                                             (30000, 64, 0.5, 0.6, 4), (9000, 40, 0.5, 0.97, 8),
                                             (70000, 256, 0.5, 0.09, 2)])
def test_exact_mode_matches_oracle_scrimp(mp, oracle_lib, n, w, ez, frac, seed):
    """The reference's SCRIMP semantics: the GPU evaluates exactly the oracle's
    first s_size diagonals of the seeded order (s_size = 1 included), so the
    partial profiles agree with or_scrimp itself; coverage is s_size / total.
    Below 9% of the diagonals that is k_diag_join (one diagonal per lane), from
    9% on k_join_masked over the bands that hold a chosen diagonal."""
    g = np.random.default_rng(seed)
    x = np.cumsum(g.standard_normal(n))
    x[n // 5:n // 5 + 3 * w] = x[n // 5]      # a flat run: the convention inside the subset
    x[n // 2:n // 2 + w] = 2.0
    zone = mp.zone_size(w, ez)
    L = n - w + 1
    nd = L - zone - 1
    s_size = max(1, int(nd * frac))
    r = mp.scrimp(x, w, ez, s_size=s_size, seed=seed)
    assert r.coverage == s_size / nd and not r.has_left_right()
    diags, cov = mp.scrimp_diagonals(n, w, zone, s_size, seed)
    assert diags.size == s_size and cov == r.coverage and np.all(diags > zone)
    ref_mp, ref_pi, _, _, ref_cov = oracle_lib.scrimp(x, w, ez, s_size=s_size, seed=seed)
    assert ref_cov == r.coverage
    ok, rel = close(r.values, ref_mp)
    assert ok, f"exact anytime MP mismatch (max rel {rel:.3e})"
    assert np.array_equal(np.isinf(r.values), np.isinf(ref_mp))
    assert not index_mismatches(r.index, ref_pi, np.arange(L), x, x, w)
    # every reported neighbour sits on a chosen diagonal
    fin = r.index >= 0
    assert np.isin(np.abs(r.index[fin] - np.arange(L)[fin]), diags).all()


def test_exact_mode_via_cpp_default(mp, oracle_lib):
    """mprof::scrimp through the C ABI default (mpgpu_scrimp) is the exact mode."""
    x = np.cumsum(np.random.default_rng(7).standard_normal(8000))
    r = mp.scrimp(x, 40, 0.5, s_size=777, seed=2)
    ref_mp = oracle_lib.scrimp(x, 40, 0.5, s_size=777, seed=2)[0]
    assert close(r.values, ref_mp)[0] and r.coverage == 777 / (8000 - 40 + 1 - 20 - 1)


def test_masked_bands_and_per_lane_diagonals_give_the_same_profile(mp, tmp_path):
    """The two exact-mode kernels on one dense set (30% of the diagonals, flat
    runs included): k_join_masked in this process, k_diag_join in a child
    process (MPGPU_MASK_MIN_DENSITY=2 is read once per process). Same values
    within the parity tolerance, same neighbours up to near-ties."""
    import os
    import subprocess
    import sys
    n, w, ez, seed = 1 << 17, 128, 0.5, 13
    x = np.cumsum(np.random.default_rng(21).standard_normal(n))
    x[3000:3000 + 4 * w] = x[3000]
    x[90000:90000 + 2 * w] = -1.5
    nd = n - w + 1 - mp.zone_size(w, ez) - 1
    s_size = int(0.3 * nd)
    np.save(tmp_path / "x.npy", x)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    child = (f"import sys, numpy as np; sys.path.insert(0, {root!r}); import paper_1904_12626_b200 as mp; "
             f"x = np.load({str(tmp_path / 'x.npy')!r}); "
             f"r = mp.scrimp(x, {w}, {ez}, s_size={s_size}, seed={seed}); "
             f"np.savez({str(tmp_path / 'lane.npz')!r}, v=r.values, i=r.index)")
    env = dict(os.environ, MPGPU_MASK_MIN_DENSITY="2")
    subprocess.run([sys.executable, "-c", child], check=True, env=env, timeout=600)
    lane = np.load(tmp_path / "lane.npz")
    r = mp.scrimp(x, w, ez, s_size=s_size, seed=seed)
    ok, rel = close(r.values, lane["v"])
    assert ok, f"masked bands vs per-lane diagonals: MP differs (max rel {rel:.3e})"
    assert not index_mismatches(r.index, lane["i"], np.arange(r.values.size), x, x, w)
    assert np.array_equal(np.isinf(r.values), np.isinf(lane["v"]))
