"""The reference's C++ API as a drop-in: a caller compiled against
include/mprof/profile.hpp and linked to libmprof_b200.so (GPU)."""
import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from tests.parity import close, index_mismatches

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    gxx = shutil.which("g++")
    libdir = os.path.join(ROOT, "paper_1904_12626_b200")
    out = str(tmp_path_factory.mktemp("cpp") / "dropin_example")
    r = subprocess.run([gxx, "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp"), "-L" + libdir,
                        "-lmprof_b200", "-Wl,-rpath," + libdir, "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def _run(exe, tmp_path, a, w, ez, mode="stomp", b=None, extra=()):
    inp = tmp_path / "a.f64"
    a.astype(np.float64).tofile(inp)
    args = [exe, str(inp), str(w), str(ez), str(tmp_path / "out"), mode, *map(str, extra)]
    if b is not None:
        bp = tmp_path / "b.f64"
        b.astype(np.float64).tofile(bp)
        args.append(str(bp))
    r = subprocess.run(args, capture_output=True, text=True)
    info = json.loads(r.stdout.strip().splitlines()[-1])
    res = {k: np.fromfile(tmp_path / f"out.{k}", dtype=np.float64 if k == "mp" else np.int64)
           for k in ("mp", "pi", "left", "right")} if r.returncode == 0 else None
    return r.returncode, info, res


def test_cpp_stomp_self_join(exe, tmp_path, oracle_lib):
    x = np.cumsum(np.random.default_rng(8).standard_normal(3000))
    rc, info, res = _run(exe, tmp_path, x, 64, 0.5)
    assert rc == 0 and info["size"] == x.size - 63 and info["zone"] == 32
    assert info["mode"] == "stomp" and info["progress_calls"] >= 1
    ref = oracle_lib.stomp(x, None, 64, 0.5, n_workers=4)
    assert close(res["mp"], ref[0])[0]
    rows = np.arange(res["mp"].size)
    assert not index_mismatches(res["pi"], ref[1], rows, x, x, 64)
    assert not index_mismatches(res["left"], ref[2], rows, x, x, 64)
    assert not index_mismatches(res["right"], ref[3], rows, x, x, 64)


def test_cpp_scrimp_and_ab(exe, tmp_path, oracle_lib):
    g = np.random.default_rng(9)
    x = np.cumsum(g.standard_normal(2000))
    rc, info, res = _run(exe, tmp_path, x, 50, 0.25, "scrimp")
    assert rc == 0 and info["mode"] == "scrimp"
    ref = oracle_lib.stomp(x, None, 50, 0.25)
    assert close(res["mp"], ref[0])[0]
    y = np.cumsum(g.standard_normal(900))
    rc, info, res = _run(exe, tmp_path, x, 50, 0.5, "ab", y)
    assert rc == 0 and info["join"] == "ab" and info["zone"] == 0
    ref = oracle_lib.stomp(x, y, 50)
    assert close(res["mp"], ref[0])[0]
    assert res["left"].size == 0 and res["right"].size == 0


def test_cpp_errors_map_to_reference_exceptions(exe, tmp_path):
    x = np.cumsum(np.random.default_rng(10).standard_normal(100))
    rc, info, _ = _run(exe, tmp_path, x, 200, 0.5)
    assert rc == 2 and info["error"] == "ParameterError"
    rc, info, _ = _run(exe, tmp_path, x[:3], 4, 0.5)
    assert rc == 2 and "too short" in info["what"]
    bad = x.copy()
    bad[17] = np.nan
    rc, info, _ = _run(exe, tmp_path, bad, 8, 0.5)
    assert rc == 2 and "not finite" in info["what"]


def test_cpp_scrimp_anytime(exe, tmp_path, oracle_lib):
    """mprof::scrimp with s_size (profile.hpp:87-89): exactly
    s_size diagonals in SCRIMP's seeded order, coverage = s_size / all
    diagonals, left/right empty, values equal the oracle's own SCRIMP run."""
    import paper_1904_12626_b200 as mp
    x = np.cumsum(np.random.default_rng(12).standard_normal(20000))
    w, ez, seed = 64, 0.5, 4
    zone = mp.zone_size(w, ez)
    L = x.size - w + 1
    nd = L - zone - 1
    s_size = nd // 5
    rc, info, res = _run(exe, tmp_path, x, w, ez, "anytime", extra=(s_size, seed))
    assert rc == 0 and info["mode"] == "scrimp" and info["coverage"] == s_size / nd
    assert res["left"].size == 0 and res["right"].size == 0
    ref_mp, ref_pi, _, _, ref_cov = oracle_lib.scrimp(x, w, ez, s_size=s_size, seed=seed)
    assert ref_cov == info["coverage"]
    assert close(res["mp"], ref_mp)[0]
    assert not index_mismatches(res["pi"], ref_pi, np.arange(L), x, x, w)


def test_cpp_simple_and_mstomp(exe, tmp_path, oracle_lib):
    """mprof::simple_join / mprof::mstomp (profile.hpp:91-100) from a C++ caller."""
    from tests.parity import mstomp_mismatches, raw_index_mismatches
    g = np.random.default_rng(13)
    x = np.cumsum(g.standard_normal((3, 1500)), axis=1)
    w = 32
    rc, info, res = _run(exe, tmp_path, x.ravel(), w, 0.5, "simple", extra=(3,))
    assert rc == 0 and info["mode"] == "simple" and info["dims"] == 3 and info["zone"] == 16
    ref = oracle_lib.simple_join(x, None, w, 0.5, n_workers=4)
    assert close(res["mp"], ref[0])[0]
    assert not raw_index_mismatches(res["pi"], ref[1], np.arange(ref[0].size), x, x, w)
    y = np.cumsum(g.standard_normal((3, 700)), axis=1)
    by = tmp_path / "y.f64"
    y.tofile(by)
    rc, info, res = _run(exe, tmp_path, x.ravel(), w, 0.5, "simple", extra=(3, by))
    assert rc == 0 and info["join"] == "ab" and res["left"].size == 0
    ref = oracle_lib.simple_join(x, y, w)
    assert close(res["mp"], ref[0])[0]
    # mstomp with a must dim and an excluded dim
    inp = tmp_path / "m.f64"
    x.tofile(inp)
    args = [exe, str(inp), str(w), "0.5", str(tmp_path / "mo"), "mstomp", "3", "2", "0"]
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    L = x.shape[1] - w + 1
    got = tuple(np.fromfile(tmp_path / f"mo.{k}", dtype=np.float64 if k == "mp" else np.int64)
                .reshape(3, L) for k in ("mp", "pi", "dim"))
    ref = oracle_lib.mstomp(x, w, 0.5, (2,), (0,), n_workers=4)
    assert not mstomp_mismatches(got, ref, x, w, (2,), (0,))
    # overlapping must / exc -> ParameterError
    args[-2:] = ["1", "1"]
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 2 and "ParameterError" in r.stdout


@pytest.fixture(scope="module")
def prim_exe(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    gxx = shutil.which("g++")
    libdir = os.path.join(ROOT, "paper_1904_12626_b200")
    out = str(tmp_path_factory.mktemp("cpp") / "primitives_example")
    r = subprocess.run([gxx, "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "primitives_example.cpp"), "-L" + libdir,
                        "-lmprof_b200", "-Wl,-rpath," + libdir, "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.parametrize("n,w,q,zone", [(5000, 64, 777, 32), (4096, 4, 0, 1), (3000, 300, 2700, 150)])
def test_cpp_primitives_vs_oracle(prim_exe, tmp_path, oracle_lib, n, w, q, zone):
    """rolling_mean_std (K1 on the GPU), is_flat_std, mass_distance_profile (K6),
    apply_exclusion_zone[_inplace], znorm_dist_from_qt and merge_min called from
    C++ through the reference signatures, against the oracle's restatements."""
    g = np.random.default_rng(n + w)
    x = np.cumsum(g.standard_normal(n))
    x[1000:1400] = 3.25  # flat run: sd == 0 exactly, is_flat_std true
    inp = tmp_path / "x.f64"
    x.tofile(inp)
    r = subprocess.run([prim_exe, str(inp), str(w), str(q), str(zone), str(tmp_path / "o")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    info = json.loads(r.stdout.strip().splitlines()[-1])
    L = n - w + 1
    rd = lambda k, t=np.float64: np.fromfile(tmp_path / f"o.{k}", dtype=t)  # noqa: E731
    mu, sd = oracle_lib.rolling_mean_std(x, w)
    gm, gs = rd("means"), rd("stds")
    assert gm.size == L and info["size"] == L and info["window"] == w
    scale = np.maximum(1.0, np.abs(mu))
    assert np.max(np.abs(gm - mu) / scale) <= 1e-12
    flat = sd == 0.0
    assert np.array_equal(gs == 0.0, flat) and info["flats"] == int(flat.sum())
    assert np.max(np.abs(gs[~flat] - sd[~flat]) / sd[~flat]) <= 1e-12
    ref = oracle_lib.mass_distance_profile(x[q:q + w], x, -1, 0)
    assert close(rd("mass"), ref, rel=1e-9, abs_=1e-9)[0]
    assert rd("mass")[q] == 0.0  # exact self-match
    ex = oracle_lib.apply_exclusion_zone(ref.copy(), q, zone)
    got_ex = rd("excl")
    assert np.array_equal(np.isinf(got_ex), np.isinf(ex)) and info["inplace_same"]
    assert int(np.isinf(got_ex).sum()) == min(L - 1, q + zone) - max(0, q - zone) + 1
    # znorm_dist_from_qt against the oracle's restatement on the same QT and
    # statistics (the raw-QT formula itself carries cancellation error, so it
    # is compared formula to formula), and loosely against the exact distances
    qt, qraw = rd("qt"), rd("qtraw")
    want = np.array([oracle_lib.znorm_dist_from_qt(v, w, gm[q], gs[q], gm[i], gs[i])
                     for i, v in enumerate(qraw)])
    # the two compilers may contract qt - w mu_a mu_b differently (FMA): bound
    # the d^2 difference by a few ulps of the cancelling terms
    eps = np.finfo(np.float64).eps
    with np.errstate(divide="ignore", invalid="ignore"):
        d2err = 16 * eps * (np.abs(qraw) + w * np.abs(gm[q] * gm)) / (gs[q] * gs)
    tol = np.where(np.isfinite(d2err), np.sqrt(np.abs(d2err)), 0.0) + 1e-9 * np.abs(want)
    assert np.all(np.abs(qt - want) <= tol + 1e-12)
    far = ref > 1.0
    assert close(qt[far], ref[far], rel=1e-3, abs_=1e-3)[0]
    mv, mi = rd("merged_v"), rd("merged_i", np.int64)
    fin = np.isfinite(got_ex)
    assert np.array_equal(mv[fin], got_ex[fin]) and np.all(mi[fin] == q)
    assert np.allclose(mv[~fin], rd("mass")[~fin] + 0.5) and np.all(mi[~fin] == q + 1)
    assert info["merge_len_error"] and info["window_error"] and info["zone_50_half"] == 25
    assert info["query_index"] == q
