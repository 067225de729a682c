"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/liboracle.so`` (a plain-C restatement of the
reference hot path, see ``mprof_oracle.h``) and ``oracle/_ref/libref_types.so``
(the reference's own ``TimeSeries`` constructor, compiled from
/root/reference/proj/src/types.cpp by ``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU baseline /
``--impl reference`` arm may import this package. The product package
``paper_1904_12626_b200`` never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_REF_LIB = os.path.join(_HERE, "_ref", "libref_types.so")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)
_lib = None
_ref = None


def build() -> None:
    """Compile liboracle.so (and _ref/ when the reference tree is present)."""
    r = subprocess.run(["make", "-s", "-C", _HERE], capture_output=True, text=True)
    sys.stderr.write(r.stdout + r.stderr)  # keep stdout clean for JSON-line tools
    if r.returncode != 0:
        raise RuntimeError("oracle build failed")


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        lib = ctypes.CDLL(_LIB)
        lib.or_zone_size.restype = ctypes.c_int64
        lib.or_zone_size.argtypes = [ctypes.c_int64, ctypes.c_double]
        lib.or_is_flat_std.restype = ctypes.c_int
        lib.or_is_flat_std.argtypes = [ctypes.c_double, ctypes.c_double]
        lib.or_rolling_mean_std.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _dp, _dp, ctypes.c_int]
        lib.or_znorm_dist_from_qt.restype = ctypes.c_double
        lib.or_znorm_dist_from_qt.argtypes = [ctypes.c_double, ctypes.c_int64] + [ctypes.c_double] * 4
        lib.or_sliding_dot_direct.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp]
        lib.or_brute_force_mp.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_double, _dp, _ip, _ip, _ip, ctypes.c_int]
        lib.or_brute_force_rows.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_double, _ip, ctypes.c_int64, _dp, _ip, _ip, _ip,
                                            ctypes.c_int]
        lib.or_stomp.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                 ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _dp, _ip, _ip, _ip]
        lib.or_scrimp.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                                  ctypes.c_uint64, _dp, _ip, _ip, _ip, _dp]
        lib.or_scrimp_diagonals.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _ip, ctypes.c_int64,
                                            _dp, _ip, ctypes.c_int]
        lib.or_mass_distance_profile.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64,
                                                 ctypes.c_int64, _dp, ctypes.c_int]
        lib.or_apply_exclusion_zone.restype = None
        lib.or_apply_exclusion_zone.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        lib.or_merge_min.restype = None
        lib.or_merge_min.argtypes = [_dp, _ip, _dp, ctypes.c_int64, ctypes.c_int64]
        lib.or_raw_norms.restype = None
        lib.or_raw_norms.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _dp]
        lib.or_raw_sq_term.restype = ctypes.c_double
        lib.or_raw_sq_term.argtypes = [ctypes.c_double] * 3
        lib.or_raw_distance_from_terms.restype = ctypes.c_double
        lib.or_raw_distance_from_terms.argtypes = [ctypes.c_double] * 2
        lib.or_raw_direct.restype = ctypes.c_double
        lib.or_raw_direct.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        lib.or_raw_distance_profile.argtypes = [_dp, _dp, ctypes.c_int64, ctypes.c_int64,
                                                ctypes.c_int64, _dp]
        lib.or_simple_join.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int64, _dp, _ip, _ip, _ip]
        lib.or_simple_brute.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_double, _dp, _ip, ctypes.c_int]
        lib.or_mstomp.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                  _ip, ctypes.c_int64, _ip, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_int64, ctypes.c_int64, _dp, _ip, _ip]
        lib.or_mstomp_dim_order.restype = ctypes.c_int64
        lib.or_mstomp_dim_order.argtypes = [ctypes.c_int64, _ip, ctypes.c_int64, _ip, ctypes.c_int64,
                                            _ip, _ip]
        lib.or_mstomp_select.restype = None
        lib.or_mstomp_select.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _ip, _ip, _dp]
        _lib = lib
    return _lib


def _d(x):
    return x.ctypes.data_as(_dp) if x is not None else None


def _i(x):
    return x.ctypes.data_as(_ip) if x is not None else None


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def zone_size(window: int, fraction: float) -> int:
    z = _load().or_zone_size(int(window), float(fraction))
    if z < 0:
        raise ValueError("negative exclusion-zone fraction")
    return int(z)


def is_flat_std(sd: float, mean: float) -> bool:
    return bool(_load().or_is_flat_std(float(sd), float(mean)))


def rolling_mean_std(ts, w: int, threads: int = 1):
    ts = _f64(ts)
    L = ts.size - w + 1
    if w < 4 or L < 1:
        raise ValueError("window out of range")
    mu = np.empty(L)
    sd = np.empty(L)
    if _load().or_rolling_mean_std(_d(ts), ts.size, w, _d(mu), _d(sd), threads):
        raise ValueError("window out of range")
    return mu, sd


def znorm_dist_from_qt(qt, w, mu_a, sd_a, mu_b, sd_b) -> float:
    return float(_load().or_znorm_dist_from_qt(qt, w, mu_a, sd_a, mu_b, sd_b))


def sliding_dot_direct(q, ts):
    q, ts = _f64(q), _f64(ts)
    out = np.empty(ts.size - q.size + 1)
    if _load().or_sliding_dot_direct(_d(q), q.size, _d(ts), ts.size, _d(out)):
        raise ValueError("length mismatch")
    return out


def _alloc(L, lr=True):
    return (np.empty(L), np.empty(L, np.int64), np.empty(L, np.int64) if lr else None,
            np.empty(L, np.int64) if lr else None)


def brute_force_mp(a, b=None, w=4, ez=0.5, threads=None):
    """brute_force_mp (profile.hpp:70-73). Returns (mp, pi, left, right)."""
    a = _f64(a)
    bb = _f64(b) if b is not None else None
    La = a.size - w + 1
    mp, pi, le, ri = _alloc(La, b is None)
    rc = _load().or_brute_force_mp(_d(a), a.size, _d(bb), 0 if bb is None else bb.size, w, ez,
                                   _d(mp), _i(pi), _i(le), _i(ri), threads or default_threads())
    if rc:
        raise ValueError("invalid window / fraction")
    return mp, pi, le, ri


def brute_force_rows(a, rows, b=None, w=4, ez=0.5, threads=None):
    """Exact MP / PI / left / right at the given profile positions only."""
    a = _f64(a)
    bb = _f64(b) if b is not None else None
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    mp, pi, le, ri = _alloc(rows.size, b is None)
    rc = _load().or_brute_force_rows(_d(a), a.size, _d(bb), 0 if bb is None else bb.size, w, ez,
                                     _i(rows), rows.size, _d(mp), _i(pi), _i(le), _i(ri),
                                     threads or default_threads())
    if rc:
        raise ValueError("invalid rows / window")
    return mp, pi, le, ri


def stomp(a, b=None, w=4, ez=0.5, n_workers=1, row_begin=0, row_end=0):
    """stomp (profile.hpp:80-83). Returns (mp, pi, left, right) for the A-profile."""
    a = _f64(a)
    bb = _f64(b) if b is not None else None
    La = a.size - w + 1
    mp, pi, le, ri = _alloc(La, True)
    rc = _load().or_stomp(_d(a), a.size, _d(bb), 0 if bb is None else bb.size, w, ez, int(n_workers),
                          int(row_begin), int(row_end), _d(mp), _i(pi), _i(le), _i(ri))
    if rc:
        raise ValueError("invalid window / fraction")
    if b is not None:
        le = ri = None
    return mp, pi, le, ri


def scrimp(a, w=4, ez=0.5, s_size=0, seed=0):
    """scrimp (profile.hpp:85-89). Returns (mp, pi, left, right, coverage)."""
    a = _f64(a)
    La = a.size - w + 1
    mp, pi, le, ri = _alloc(La, True)
    cov = ctypes.c_double(0)
    rc = _load().or_scrimp(_d(a), a.size, w, ez, int(s_size), ctypes.c_uint64(seed), _d(mp), _i(pi),
                           _i(le), _i(ri), ctypes.byref(cov))
    if rc:
        raise ValueError("invalid window / fraction")
    return mp, pi, le, ri, cov.value


def scrimp_diagonals(a, w, diags, threads=None):
    """MP / PI over exactly the given diagonals (anytime-run checker)."""
    a = _f64(a)
    diags = np.ascontiguousarray(diags, dtype=np.int64)
    L = a.size - w + 1
    mp, pi = np.empty(L), np.empty(L, np.int64)
    if _load().or_scrimp_diagonals(_d(a), a.size, w, _i(diags), diags.size, _d(mp), _i(pi),
                                   threads or default_threads()):
        raise ValueError("invalid window")
    return mp, pi


def mass_distance_profile(query, ts, query_index=-1, zone=0, threads=None):
    """Exact distance profile of one query (mass_distance_profile, distance.hpp:26-33)."""
    q, ts = _f64(query), _f64(ts)
    out = np.empty(ts.size - q.size + 1)
    if _load().or_mass_distance_profile(_d(q), q.size, _d(ts), ts.size, int(query_index), int(zone),
                                        _d(out), threads or default_threads()):
        raise ValueError("window out of range")
    return out


def apply_exclusion_zone(dp, center, zone):
    dp = _f64(dp).copy()
    _load().or_apply_exclusion_zone(_d(dp), dp.size, int(center), int(zone))
    return dp


def merge_min(acc, acc_idx, dp, source_index):
    _load().or_merge_min(_d(acc), _i(acc_idx), _d(_f64(dp)), acc.size, int(source_index))


def ref_timeseries_validate(x):
    """Run the reference's own TimeSeries constructor (types.cpp:7-18).

    Returns (code, message): 0 = accepted, 2 = ParameterError. Raises
    FileNotFoundError when oracle/_ref was never built.
    """
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_LIB):
            raise FileNotFoundError(_REF_LIB)
        _ref = ctypes.CDLL(_REF_LIB)
        _ref.ref_timeseries_validate.argtypes = [_dp, ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
    x = _f64(x)
    buf = ctypes.create_string_buffer(256)
    rc = _ref.ref_timeseries_validate(_d(x), x.size, buf, 256)
    return rc, buf.value.decode()


# ---------------------------------------------------------------- MP consumers
# numpy restatements of discovery.hpp:61-79 (checkers for the GPU versions).

def fluss_arc_count(index):
    """arc_counts[i] = number of nearest-neighbour arcs strictly crossing i
    (discovery.hpp:68-70), via a +1/-1 sweep."""
    index = np.asarray(index, dtype=np.int64)
    L = index.size
    i = np.arange(L)
    ok = (index >= 0) & (index < L) & (index != i)
    lo = np.minimum(i, index)[ok]
    hi = np.maximum(i, index)[ok]
    keep = hi - lo >= 2
    diff = np.zeros(L + 1, np.int64)
    np.add.at(diff, lo[keep] + 1, 1)
    np.add.at(diff, hi[keep], -1)
    return np.cumsum(diff[:L])


def fluss_cac(arcs, window):
    """Corrected arc curve (discovery.hpp:72-74)."""
    arcs = np.asarray(arcs, dtype=np.float64)
    L = arcs.size
    i = np.arange(L, dtype=np.float64)
    ideal = 2.0 * i * (L - i) / L
    with np.errstate(divide="ignore", invalid="ignore"):
        cac = np.where(ideal > 0, arcs / ideal, 1.0)
    cac = np.clip(cac, 0.0, 1.0)
    cac[:window] = 1.0
    cac[max(0, L - window):] = 1.0
    return cac


def extract(values, k, zone, largest, stop_at):
    """Repeated arg-extreme with +-zone masking (find_discord / fluss_extract)."""
    v = np.array(values, dtype=np.float64)
    out = []
    for _ in range(k):
        fin = np.isfinite(v)
        if not fin.any():
            break
        if largest:
            j = int(np.argmax(np.where(fin, v, -np.inf)))
            if not v[j] > stop_at:
                break
        else:
            j = int(np.argmin(np.where(fin, v, np.inf)))
            if not v[j] < stop_at:
                break
        out.append((j, float(v[j])))
        v[max(0, j - zone):j + zone + 1] = np.inf if not largest else -np.inf
    return out


# ---------------------------------------------------------------- multivariate
# SiMPle / mSTOMP (profile.hpp:91-100). Multivariate series are (dims, n)
# arrays, passed dim-major.

def _mts(x):
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[None, :]
    return np.ascontiguousarray(x)


RAW_SNAP = 1e-12  # OR_RAW_SNAP (mprof_oracle.h)


def raw_distance_from_terms(dsq, scale) -> float:
    return float(_load().or_raw_distance_from_terms(float(dsq), float(scale)))


def raw_sq_term(sa, sb, qt) -> float:
    return float(_load().or_raw_sq_term(float(sa), float(sb), float(qt)))


def raw_distance_profile(query, mts):
    """raw_distance_profile (distance.hpp:44-49): query (dims, w) vs every window."""
    q, x = _mts(query), _mts(mts)
    if q.shape[0] != x.shape[0]:
        raise ValueError("dimension mismatch")
    out = np.empty(x.shape[1] - q.shape[1] + 1)
    if _load().or_raw_distance_profile(_d(q), _d(x), x.shape[1], x.shape[0], q.shape[1], _d(out)):
        raise ValueError("window out of range")
    return out


def raw_direct(a, i, b, j, w) -> float:
    a, b = _mts(a), _mts(b)
    return float(_load().or_raw_direct(_d(a), a.shape[1], _d(b), b.shape[1], a.shape[0], w, i, j))


def simple_join(a, b=None, w=4, ez=0.5, n_workers=1, row_begin=0, row_end=0):
    """simple (profile.hpp:96-100). Returns (mp, pi, left, right); AB: left/right None."""
    a = _mts(a)
    bb = _mts(b) if b is not None else None
    if bb is not None and bb.shape[0] != a.shape[0]:
        raise ValueError("dimension mismatch")
    La = a.shape[1] - w + 1
    mp, pi, le, ri = _alloc(La, True)
    rc = _load().or_simple_join(_d(a), a.shape[1], _d(bb), 0 if bb is None else bb.shape[1],
                                a.shape[0], w, ez, int(n_workers), int(row_begin), int(row_end),
                                _d(mp), _i(pi), _i(le), _i(ri))
    if rc:
        raise ValueError("invalid window / fraction")
    if b is not None:
        le = ri = None
    return mp, pi, le, ri


def simple_brute(a, b=None, w=4, ez=0.5, threads=None):
    a = _mts(a)
    bb = _mts(b) if b is not None else None
    La = a.shape[1] - w + 1
    mp, pi = np.empty(La), np.empty(La, np.int64)
    if _load().or_simple_brute(_d(a), a.shape[1], _d(bb), 0 if bb is None else bb.shape[1],
                               a.shape[0], w, ez, _d(mp), _i(pi), threads or default_threads()):
        raise ValueError("invalid window")
    return mp, pi


def _dimlist(v):
    return np.ascontiguousarray(list(v) if v is not None else [], dtype=np.int64)


def mstomp(x, w, ez=0.5, must_dims=(), exc_dims=(), n_workers=1, row_begin=0, row_end=0):
    """mstomp (profile.hpp:91-94). Returns (values, index, dim_order), each (dims, L)."""
    x = _mts(x)
    d, n = x.shape
    L = n - w + 1
    must, exc = _dimlist(must_dims), _dimlist(exc_dims)
    mp = np.empty((d, L))
    pi = np.empty((d, L), np.int64)
    do = np.empty((d, L), np.int64)
    rc = _load().or_mstomp(_d(x), n, d, w, ez, _i(must), must.size, _i(exc), exc.size,
                           int(n_workers), int(row_begin), int(row_end), _d(mp), _i(pi), _i(do))
    if rc == -2:
        raise ValueError("invalid must / exc dimensions")
    if rc:
        raise ValueError("invalid window / fraction")
    return mp, pi, do


def mstomp_dim_order(dims, must_dims=(), exc_dims=()):
    must, exc = _dimlist(must_dims), _dimlist(exc_dims)
    order = np.empty(max(dims, 1), np.int64)
    nm = ctypes.c_int64(0)
    c = _load().or_mstomp_dim_order(dims, _i(must), must.size, _i(exc), exc.size, _i(order),
                                    ctypes.byref(nm))
    if c < 0:
        raise ValueError("invalid must / exc dimensions")
    return order[:c], int(nm.value)


def mstomp_select(dist, n_must, order):
    """Per-cell selection: (slot dims, prefix means) for admissible distances
    given in `order` (positions into order)."""
    dist = _f64(dist)
    order = np.ascontiguousarray(order, dtype=np.int64)
    slot = np.empty(dist.size, np.int64)
    pk = np.empty(dist.size)
    _load().or_mstomp_select(_d(dist), dist.size, int(n_must), _i(order), _i(slot), _d(pk))
    return slot, pk
