"""The five BASELINE.json configs at full size on the GPU.

C1 is checked row-for-row elsewhere (test_gpu_parity.py). Here: C2, C3 (both
directions) and the headline C4 against the FULL CPU STOMP oracle on every
row (MP, PI, left, right), plus the planted
motifs / discord and the constant segments; C5 (n = 2^23) against the
sampled-row brute-force oracle (256 seeded rows, the first and last zone + 2
rows) and size-independent properties on every row (zone law, left < i <
right, MP = distance to PI recomputed exactly on a random subset).
"""
import numpy as np
import pytest

from tests.parity import close, exact_dist, index_mismatches

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_12626_b200 as mp
    mp.lib()
    return mp


def _sample_rows(L, zone, n_random, seed, extra=()):
    g = np.random.default_rng(seed)
    rows = set(g.choice(L, size=min(n_random, L), replace=False).tolist())
    rows.update(range(min(zone + 2, L)))
    rows.update(range(max(0, L - zone - 2), L))
    rows.update(int(r) for r in extra if 0 <= r < L)
    return np.array(sorted(rows), dtype=np.int64)


def _check_rows(got_mp, got_pi, got_left, got_right, rows, ref, x, y, m, self_join):
    ok, rel = close(got_mp[rows], ref[0])
    assert ok, f"MP mismatch on sampled rows (max rel {rel:.3e})"
    assert not index_mismatches(got_pi[rows], ref[1], rows, x, y, m)
    if self_join:
        assert not index_mismatches(got_left[rows], ref[2], rows, x, y, m)
        assert not index_mismatches(got_right[rows], ref[3], rows, x, y, m)


def _properties(r, x, m, zone, n_check=1500, seed=0):
    L = r.values.size
    i = np.arange(L)
    fin = np.isfinite(r.values)
    assert np.all(np.abs(r.index[fin] - i[fin]) > zone)          # zone law
    assert np.all(r.left_index[r.left_index >= 0] < i[r.left_index >= 0])
    assert np.all(r.right_index[r.right_index >= 0] > i[r.right_index >= 0])
    assert np.all((r.index == r.left_index) | (r.index == r.right_index))
    g = np.random.default_rng(seed)
    for k in g.choice(np.flatnonzero(fin), size=min(n_check, fin.sum()), replace=False):
        d = exact_dist(x, int(k), x, int(r.index[k]), m)
        assert abs(d - r.values[k]) <= 1e-6 * max(d, 1.0), (k, d, r.values[k])


def test_c2_full_oracle_and_planted(mp, oracle_lib):
    from paper_1904_12626_b200 import datasets
    c = datasets.c2()
    r = mp.stomp(c.a, None, c.window, c.ez)
    ref = oracle_lib.stomp(c.a, None, c.window, c.ez, n_workers=oracle_lib.default_threads())
    ok, rel = close(r.values, ref[0])
    assert ok, f"C2 MP max rel {rel:.3e}"
    rows = np.arange(r.values.size)
    for got, exp in ((r.index, ref[1]), (r.left_index, ref[2]), (r.right_index, ref[3])):
        assert not index_mismatches(got, exp, rows, c.a, c.a, c.window)
    # planted motif pairs find each other; the planted discord tops the profile
    for s1, s2, _ in c.planted["pairs"]:
        assert abs(int(r.index[s1]) - s2) <= 2 and r.values[s1] < 2.0
    d = c.planted["discord"]
    top = int(np.argmax(np.where(np.isfinite(r.values), r.values, -1)))
    assert abs(top - d) <= c.window


def _full_oracle_check(r, ref, x, y, m, self_join, what):
    ok, rel = close(r.values, ref[0])
    assert ok, f"{what} MP max rel {rel:.3e}"
    rows = np.arange(r.values.size)
    pairs = [("index", r.index, ref[1])]
    if self_join:
        pairs += [("left", r.left_index, ref[2]), ("right", r.right_index, ref[3])]
    for name, got, exp in pairs:
        bad = index_mismatches(got, exp, rows, x, y, m)
        assert not bad, f"{what} {name}: {len(bad)} unexplained mismatches, e.g. {bad[:3]}"


def test_c3_ab_full_both_directions(mp, oracle_lib):
    from paper_1904_12626_b200 import datasets
    c = datasets.c3()
    pa, pb = mp.stomp_ab(c.a, c.b, c.window)
    nw = oracle_lib.default_threads()
    # oracle stomp(a, b): the profile of A against B (rows over B)
    ref_a = oracle_lib.stomp(c.a, c.b, c.window, 0.0, n_workers=nw)
    ref_b = oracle_lib.stomp(c.b, c.a, c.window, 0.0, n_workers=nw)
    _full_oracle_check(pa, ref_a, c.a, c.b, c.window, False, "C3 A|B")
    _full_oracle_check(pb, ref_b, c.b, c.a, c.window, False, "C3 B|A")
    assert np.all(np.isfinite(pa.values)) and np.all(np.isfinite(pb.values))


def test_c4_ecg_full_oracle_and_flat(mp, oracle_lib):
    """The headline config on every one of its 1,048,321 rows against the full
    oracle STOMP (about 1.1e12 cell evaluations: ~6 min on 16 host threads)."""
    from paper_1904_12626_b200 import datasets
    c = datasets.c4()
    r = mp.stomp(c.a, None, c.window, c.ez)
    ref = oracle_lib.stomp(c.a, None, c.window, c.ez, n_workers=oracle_lib.default_threads())
    _full_oracle_check(r, ref, c.a, c.a, c.window, True, "C4")
    # every window wholly inside a constant run has MP 0 (flat-vs-flat convention)
    for s in c.planted["flat_segments"]:
        inside = np.arange(s, s + 5000 - c.window + 1)
        assert np.all(r.values[inside] == 0.0)
    _properties(r, c.a, c.window, c.zone)


def test_c5_sampled(mp, oracle_lib):
    from paper_1904_12626_b200 import datasets
    c = datasets.c5()
    r = mp.stomp(c.a, None, c.window, c.ez)
    rows = _sample_rows(r.values.size, c.zone, 256, 5)
    ref = oracle_lib.brute_force_rows(c.a, rows, None, c.window, c.ez)
    _check_rows(r.values, r.index, r.left_index, r.right_index, rows, ref, c.a, c.a, c.window, True)
    _properties(r, c.a, c.window, c.zone, n_check=500)
