"""MP consumers on the GPU (discovery.hpp:61-79): FLUSS arc count / CAC /
segment extraction and discords, against the oracle's numpy restatements, on
the BASELINE configs' profiles (planted discord in C2, flat segments in C4)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_12626_b200 as mp
    mp.lib()
    return mp


def test_fluss_matches_oracle(mp, oracle_lib):
    g = np.random.default_rng(51)
    # regime change: two different random processes back to back
    x = np.r_[np.cumsum(g.standard_normal(20000)), np.sin(np.arange(20000) / 7.0) * 5
              + g.standard_normal(20000)]
    w = 100
    prof = mp.stomp(x, None, w, 0.5)
    arcs, cac = mp.fluss(prof.index, w)
    ref_arcs = oracle_lib.fluss_arc_count(prof.index)
    assert np.array_equal(arcs, ref_arcs)
    assert np.allclose(cac, oracle_lib.fluss_cac(ref_arcs, w), rtol=0, atol=1e-15)
    segs, trunc = mp.fluss_extract(cac, 3, w)
    ref = oracle_lib.extract(cac, 3, int(5 * w), False, 1.0)
    assert segs == [j for j, _ in ref]
    assert abs(segs[0] - 20000) < 1000  # the regime change is the first cut


def test_discords_match_oracle_and_find_planted(mp, oracle_lib):
    from paper_1904_12626_b200 import datasets
    c = datasets.c2()
    prof = mp.stomp(c.a, None, c.window, c.ez)
    got, trunc = mp.find_discord(prof, 5)
    ref = oracle_lib.extract(prof.values, 5, prof.exclusion_zone, True, -np.inf)
    assert [j for j, _ in got] == [j for j, _ in ref] and not trunc
    assert abs(got[0][0] - c.planted["discord"]) <= c.window
    # truncation: more discords than the masked profile can hold
    x = np.cumsum(np.random.default_rng(52).standard_normal(600))
    p = mp.stomp(x, None, 50, 0.5)
    many, trunc = mp.find_discord(p, 100)
    assert trunc and len(many) == len(oracle_lib.extract(p.values, 100, p.exclusion_zone, True, -np.inf))


def test_fluss_scan_tiles_match_oracle(mp, oracle_lib):
    """Arc counts across several 4096-window scan tiles (and ragged tails) equal
    the oracle's sweep exactly; the CAC matches to the last bit."""
    g = np.random.default_rng(44)
    for L in (4095, 4096, 4097, 3 * 4096 + 17, (1 << 20) + 5):
        pi = g.integers(-1, L, L).astype(np.int64)
        arcs, cac = mp.fluss(pi, 64)
        ref = oracle_lib.fluss_arc_count(pi)
        assert np.array_equal(arcs, ref), L
        assert np.array_equal(cac, oracle_lib.fluss_cac(ref, 64)), L


def test_fluss_near_arcs_and_tiny_lengths(mp, oracle_lib):
    """Arcs to the adjacent windows (no interior), to i +- 2 (one interior
    window, both ends next to each other), self and out-of-range pointers, and
    lengths 1-3; the near end of every arc is taken in the scan passes and the
    far end by the atomic pass."""
    g = np.random.default_rng(45)
    for L in (1, 2, 3, 5, 4096 + 3):
        for kind in range(4):
            i = np.arange(L)
            off = g.choice([-2, -1, 0, 1, 2], L) if kind == 0 else np.full(L, (-2, 2, 1)[kind - 1])
            pi = (i + off).astype(np.int64)
            pi[pi >= L] = -1
            arcs, cac = mp.fluss(pi, 1)
            ref = oracle_lib.fluss_arc_count(pi)
            assert np.array_equal(arcs, ref), (L, kind)
            assert np.array_equal(cac, oracle_lib.fluss_cac(ref, 1)), (L, kind)
