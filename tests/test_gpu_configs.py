"""The five BASELINE.json configs at full size on the GPU.

C1 is checked row-for-row elsewhere (test_gpu_parity.py). Here: C2 against
the full CPU STOMP oracle (plus the planted motifs / discord), C3-C5 against
the sampled-row brute-force oracle (exact MP / PI / left / right on seeded
rows, the first and last zone rows and every flat-adjacent row), and
size-independent properties on every row (zone law, left < i < right,
MP = distance to PI recomputed exactly on a random subset).
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


def test_c3_ab_sampled(mp, oracle_lib):
    from paper_1904_12626_b200 import datasets
    c = datasets.c3()
    pa, pb = mp.stomp_ab(c.a, c.b, c.window)
    for prof, x, y in ((pa, c.a, c.b), (pb, c.b, c.a)):
        rows = _sample_rows(prof.values.size, 0, 192, 3)
        ref = oracle_lib.brute_force_rows(x, rows, y, c.window)
        ok, rel = close(prof.values[rows], ref[0])
        assert ok, f"C3 MP max rel {rel:.3e}"
        assert not index_mismatches(prof.index[rows], ref[1], rows, x, y, c.window)
        assert np.all(np.isfinite(prof.values))


def test_c4_ecg_sampled_and_flat(mp, oracle_lib):
    from paper_1904_12626_b200 import datasets
    c = datasets.c4()
    r = mp.stomp(c.a, None, c.window, c.ez)
    L = r.values.size
    flats = c.planted["flat_segments"]
    extra = []
    for s in flats:  # windows entering / inside / leaving each constant run
        extra += [s - c.window, s - 1, s, s + 5000 - c.window, s + 5000 - c.window + 1, s + 5000]
    rows = _sample_rows(L, c.zone, 192, 4, extra)
    ref = oracle_lib.brute_force_rows(c.a, rows, None, c.window, c.ez)
    _check_rows(r.values, r.index, r.left_index, r.right_index, rows, ref, c.a, c.a, c.window, True)
    # every window wholly inside a constant run has MP 0 (flat-vs-flat convention)
    for s in flats:
        inside = np.arange(s, s + 5000 - c.window + 1)
        assert np.all(r.values[inside] == 0.0)
    _properties(r, c.a, c.window, c.zone)


def test_c5_sampled(mp, oracle_lib):
    from paper_1904_12626_b200 import datasets
    c = datasets.c5()
    r = mp.stomp(c.a, None, c.window, c.ez)
    rows = _sample_rows(r.values.size, c.zone, 48, 5)
    ref = oracle_lib.brute_force_rows(c.a, rows, None, c.window, c.ez)
    _check_rows(r.values, r.index, r.left_index, r.right_index, rows, ref, c.a, c.a, c.window, True)
    _properties(r, c.a, c.window, c.zone, n_check=500)
