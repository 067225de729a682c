"""K1 (window statistics) through its exported entry point mpgpu_rolling_stats
/ mp.rolling_stats (rolling_mean_std + is_flat_std, rolling.hpp:21-29) against
the oracle's direct two-pass statistics (<= 1e-12 relative) and the SPEC.md
known answers (tests/golden/spec_kat.json), at sizes up to the
C5 series (n = 2^23)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_12626_b200 as mp
    mp.lib()
    return mp


def _gpu_stats(mp, x, w):
    import torch
    mu, sd = mp.rolling_stats(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda(), w)
    return mu.cpu().numpy(), sd.cpu().numpy()


def test_spec_known_answers(mp):
    kat = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_kat.json")))
    cases = kat["rolling_mean_std"]
    assert len(cases) >= 2
    for c in cases:
        mu, sd = _gpu_stats(mp, np.array(c["ts"], dtype=np.float64), c["w"])
        assert np.allclose(mu, c["means"], rtol=0, atol=1e-15), (c, mu)
        assert np.allclose(sd, c["stds"], rtol=0, atol=1e-15), (c, sd)


@pytest.mark.parametrize("n,w", [(1024, 64), (100000, 4), (1 << 20, 256), (1 << 23, 128), (70000, 9000)])
def test_rolling_stats_vs_oracle(mp, oracle_lib, n, w):
    g = np.random.default_rng(n ^ w)
    x = np.cumsum(g.standard_normal(n)) + 1e3  # offset: large means, the cancellation case
    x[n // 3:n // 3 + 2 * w] = x[n // 3]       # a flat run (sd floored to 0)
    x[n // 2:n // 2 + w] += 1e-13 * g.standard_normal(w)  # sub-threshold wiggle: flat as well
    mu, sd = _gpu_stats(mp, x, w)
    rmu, rsd = oracle_lib.rolling_mean_std(x, w, threads=8)
    assert mu.size == n - w + 1
    assert np.max(np.abs(mu - rmu) / np.maximum(1.0, np.abs(rmu))) <= 1e-12
    flat = rsd == 0.0
    assert flat.any() and np.array_equal(sd == 0.0, flat)
    assert np.max(np.abs(sd[~flat] - rsd[~flat]) / rsd[~flat]) <= 1e-12


def test_reversal_property(mp):
    """rolling_mean_std over a reversed series equals the reversed stats."""
    g = np.random.default_rng(5)
    x = np.cumsum(g.standard_normal(50000))
    mu, sd = _gpu_stats(mp, x, 100)
    rmu, rsd = _gpu_stats(mp, x[::-1].copy(), 100)
    assert np.allclose(rmu[::-1], mu, rtol=1e-12, atol=1e-12)
    assert np.allclose(rsd[::-1], sd, rtol=1e-12, atol=0)


@pytest.mark.parametrize("w", [4, 5, 100, 256, 513, 1000, 2049])
def test_blocked_and_per_window_kernels_agree_bit_for_bit(mp, w):
    """K1 switches kernels by series length (one thread per window below 303K
    windows, 8 windows per thread on a register window above). Both add each
    window's samples in order, so a long series and a slice of it give the
    same bits for the windows they share (also across the 512-sample chunks of
    the blocked kernel and for windows that are no multiple of 8 long)."""
    import torch
    g = np.random.default_rng(w)
    n = 400_000 + w
    x = np.cumsum(g.standard_normal(n)) * 1e3 + 1e6
    x[1000:1000 + 3 * w] = x[1000]  # a flat run
    xd = torch.from_numpy(x).cuda()
    mu_l, sd_l = mp.rolling_stats(xd, w)                      # 400,001 windows: blocked
    lo, cnt = 123_457, 50_000
    mu_s, sd_s = mp.rolling_stats(xd[lo:lo + cnt + w - 1].contiguous(), w)   # 50,000 windows: per window
    assert torch.equal(mu_l[lo:lo + cnt], mu_s) and torch.equal(sd_l[lo:lo + cnt], sd_s)
    mu_h, sd_h = mp.rolling_stats(xd[:60_000 + w - 1].contiguous(), w)
    assert torch.equal(mu_l[:60_000], mu_h) and torch.equal(sd_l[:60_000], sd_h)
    assert float(sd_l[1000]) == 0.0
