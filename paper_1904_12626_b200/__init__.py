"""B200-native exact z-normalised similarity join (matrix profile).

Python mirror of the reference's C++ hot-path API
(/root/reference/proj/include/mprof/profile.hpp:80-89): ``stomp`` and
``scrimp`` take a series, a window and an exclusion-zone fraction and return a
``MatrixProfile`` with the reference's fields and error behaviour
(ParameterError / UnsupportedError, error.hpp:9-19). Everything runs through
the C ABI of ``libmprof_b200.so`` (include/mprof_gpu.h) on sm_100a; there is
no CPU fallback — a missing library or GPU raises.

``Plan`` exposes the device-resident, sharded form (torch CUDA tensors in,
packed int64 keys out) that ``bench.py`` drives across ranks with
``torch.distributed`` (NCCL ReduceOp.MIN over the keys).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

__all__ = [
    "ParameterError", "UnsupportedError", "MatrixProfile", "zone_size", "join_cells",
    "stomp", "scrimp", "scrimp_bands", "band_diagonals", "stomp_ab", "join", "Plan",
    "distance_profiles", "mass_distance_profile", "find_discord", "fluss", "fluss_extract",
    "rolling_stats", "lib", "K_FULL_RUN", "MIN_WINDOW",
    "MultiTimeSeries", "MultiMatrixProfile", "simple_join", "mstomp",
]

K_FULL_RUN = (1 << 63) - 1   # kFullRun (profile.hpp:20-21)
MIN_WINDOW = 4               # kMinWindow (types.hpp:19-21)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("MPGPU_LIB") or os.path.join(_HERE, "libmprof_b200.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)
_PROGRESS = ctypes.CFUNCTYPE(None, ctypes.c_double, ctypes.c_void_p)

MPGPU_OK, MPGPU_EPARAM, MPGPU_EUNSUPPORTED = 0, 2, 3


class ParameterError(ValueError):
    """Invalid argument (reference ParameterError, error.hpp:9-13)."""


class UnsupportedError(ParameterError):
    """Unsupported mode combination (reference UnsupportedError, error.hpp:15-19)."""


class _JoinArgs(ctypes.Structure):
    _fields_ = [
        ("a", _dp), ("n_a", ctypes.c_int64), ("b", _dp), ("n_b", ctypes.c_int64),
        ("window", ctypes.c_int64), ("zone", ctypes.c_int64),
        ("n_gpus", ctypes.c_int32), ("devices", ctypes.POINTER(ctypes.c_int32)),
        ("mp_a", _dp), ("pi_a", _ip), ("left_a", _ip), ("right_a", _ip),
        ("mp_b", _dp), ("pi_b", _ip),
        ("progress", _PROGRESS), ("progress_ctx", ctypes.c_void_p),
    ]


class _SimpleArgs(ctypes.Structure):
    _fields_ = [
        ("a", _dp), ("n_a", ctypes.c_int64), ("b", _dp), ("n_b", ctypes.c_int64),
        ("dims", ctypes.c_int64), ("window", ctypes.c_int64), ("zone", ctypes.c_int64),
        ("device", ctypes.c_int32),
        ("mp_a", _dp), ("pi_a", _ip), ("left_a", _ip), ("right_a", _ip),
        ("mp_b", _dp), ("pi_b", _ip), ("kernel_ms", _dp),
    ]


class _MStompArgs(ctypes.Structure):
    _fields_ = [
        ("x", _dp), ("n", ctypes.c_int64), ("dims", ctypes.c_int64), ("window", ctypes.c_int64),
        ("zone", ctypes.c_int64), ("must_dims", _ip), ("n_must", ctypes.c_int64),
        ("exc_dims", _ip), ("n_exc", ctypes.c_int64), ("device", ctypes.c_int32),
        ("mp", _dp), ("pi", _ip), ("dim_order", _ip), ("kernel_ms", _dp),
    ]


def lib() -> ctypes.CDLL:
    """Load libmprof_b200.so (built in-tree by build.py). Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: run `python -m paper_1904_12626_b200.build` "
            "(the product has no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    L.mpgpu_join.argtypes = [ctypes.POINTER(_JoinArgs)]
    L.mpgpu_join.restype = ctypes.c_int
    L.mpgpu_join_timed.argtypes = [ctypes.POINTER(_JoinArgs), _dp, _dp]
    L.mpgpu_join_timed.restype = ctypes.c_int
    L.mpgpu_last_error.restype = ctypes.c_char_p
    L.mpgpu_zone_size.argtypes = [ctypes.c_int64, ctypes.c_double]
    L.mpgpu_zone_size.restype = ctypes.c_int64
    L.mpgpu_join_cells.argtypes = [ctypes.c_int64] * 4
    L.mpgpu_join_cells.restype = ctypes.c_int64
    L.mpgpu_rolling_stats.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                      ctypes.c_void_p]
    L.mpgpu_rolling_stats.restype = ctypes.c_int
    L.mpgpu_plan_create.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]
    L.mpgpu_plan_create.restype = ctypes.c_void_p
    L.mpgpu_plan_destroy.argtypes = [ctypes.c_void_p]
    L.mpgpu_plan_destroy.restype = None
    L.mpgpu_plan_prepare.argtypes = [ctypes.c_void_p]
    L.mpgpu_plan_prepare.restype = ctypes.c_int
    L.mpgpu_plan_prepare_shard.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
    L.mpgpu_plan_prepare_shard.restype = ctypes.c_int
    L.mpgpu_plan_prepare_finish.argtypes = [ctypes.c_void_p]
    L.mpgpu_plan_prepare_finish.restype = ctypes.c_int
    L.mpgpu_plan_coarse_keys.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), _ip,
                                         ctypes.POINTER(ctypes.c_void_p), _ip]
    L.mpgpu_plan_coarse_keys.restype = ctypes.c_int
    L.mpgpu_plan_run.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
    L.mpgpu_plan_run.restype = ctypes.c_int
    L.mpgpu_plan_shard_cells.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
    L.mpgpu_plan_shard_cells.restype = ctypes.c_int64
    L.mpgpu_plan_keys.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), _ip,
                                  ctypes.POINTER(ctypes.c_void_p), _ip]
    L.mpgpu_plan_keys.restype = ctypes.c_int
    L.mpgpu_plan_finalize.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 6
    L.mpgpu_plan_finalize.restype = ctypes.c_int
    L.mpgpu_plan_finalize_shard.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32] + \
        [ctypes.c_void_p] * 6
    L.mpgpu_plan_finalize_shard.restype = ctypes.c_int
    L.mpgpu_keys_min_merge.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_void_p]
    L.mpgpu_keys_min_merge.restype = ctypes.c_int
    L.mpgpu_plan_launch_count.argtypes = [ctypes.c_void_p]
    L.mpgpu_plan_launch_count.restype = ctypes.c_int64
    L.mpgpu_build_info.restype = ctypes.c_char_p
    L.mpgpu_scrimp.argtypes = [ctypes.POINTER(_JoinArgs), ctypes.c_int64, ctypes.c_uint64, _dp]
    L.mpgpu_scrimp.restype = ctypes.c_int
    L.mpgpu_scrimp_bands.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_uint64, _ip, ctypes.c_int64, _dp]
    L.mpgpu_scrimp_bands.restype = ctypes.c_int64
    L.mpgpu_scrimp_diagonals.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_uint64, _ip, ctypes.c_int64, _dp]
    L.mpgpu_scrimp_diagonals.restype = ctypes.c_int64
    L.mpgpu_scrimp_banded.argtypes = [ctypes.POINTER(_JoinArgs), ctypes.c_int64, ctypes.c_uint64, _dp]
    L.mpgpu_scrimp_banded.restype = ctypes.c_int
    L.mpgpu_plan_select_bands.argtypes = [ctypes.c_void_p, _ip, ctypes.c_int64]
    L.mpgpu_plan_select_bands.restype = ctypes.c_int
    L.mpgpu_distance_profiles.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                          ctypes.c_void_p]
    L.mpgpu_distance_profiles.restype = ctypes.c_int
    L.mpgpu_fluss.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]
    L.mpgpu_fluss.restype = ctypes.c_int
    L.mpgpu_extract.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int32, ctypes.c_double, _ip, _dp, ctypes.c_int32,
                                ctypes.c_void_p]
    L.mpgpu_extract.restype = ctypes.c_int64
    L.mpgpu_plan_attach_keys.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    L.mpgpu_plan_attach_keys.restype = ctypes.c_int
    for fn in ("mpgpu_plan_prepare_shared", "mpgpu_plan_seed_shared"):
        getattr(L, fn).argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
        getattr(L, fn).restype = ctypes.c_int
    L.mpgpu_plan_coarse_key_ptrs.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                             ctypes.POINTER(ctypes.c_void_p)]
    L.mpgpu_plan_coarse_key_ptrs.restype = ctypes.c_int
    L.mpgpu_plan_attach_coarse_keys.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    L.mpgpu_plan_attach_coarse_keys.restype = ctypes.c_int
    L.mpgpu_plan_coarse_run.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
    L.mpgpu_plan_coarse_run.restype = ctypes.c_int
    L.mpgpu_plan_reset_keys.argtypes = [ctypes.c_void_p]
    L.mpgpu_plan_reset_keys.restype = ctypes.c_int
    L.mpgpu_ipc_export.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int32]
    L.mpgpu_ipc_export.restype = ctypes.c_int
    L.mpgpu_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32]
    L.mpgpu_ipc_open.restype = ctypes.c_int
    L.mpgpu_ipc_close.argtypes = [ctypes.c_void_p, ctypes.c_int32]
    L.mpgpu_ipc_close.restype = ctypes.c_int
    L.mpgpu_stripes_granularity.argtypes = [ctypes.c_int32]
    L.mpgpu_stripes_granularity.restype = ctypes.c_int64
    L.mpgpu_stripes_create.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.POINTER(ctypes.c_int32)]
    L.mpgpu_stripes_create.restype = ctypes.c_void_p
    L.mpgpu_stripes_create_local.argtypes = [ctypes.c_int64, ctypes.c_int32,
                                             ctypes.POINTER(ctypes.c_int32),
                                             ctypes.POINTER(ctypes.c_int32)]
    L.mpgpu_stripes_create_local.restype = ctypes.c_void_p
    for fn in ("mpgpu_stripes_num_chunks", "mpgpu_stripes_chunk_bytes"):
        getattr(L, fn).argtypes = [ctypes.c_void_p]
        getattr(L, fn).restype = ctypes.c_int64
    L.mpgpu_stripes_owner.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    L.mpgpu_stripes_owner.restype = ctypes.c_int32
    L.mpgpu_stripes_export_fd.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    L.mpgpu_stripes_export_fd.restype = ctypes.c_int32
    L.mpgpu_stripes_import_fd.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32]
    L.mpgpu_stripes_import_fd.restype = ctypes.c_int
    L.mpgpu_stripes_map.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    L.mpgpu_stripes_map.restype = ctypes.c_int
    L.mpgpu_stripes_destroy.argtypes = [ctypes.c_void_p]
    L.mpgpu_stripes_destroy.restype = None
    L.mpgpu_device_pci_bus_id.argtypes = [ctypes.c_int32, ctypes.c_char_p, ctypes.c_int32]
    L.mpgpu_device_pci_bus_id.restype = ctypes.c_int32
    L.mpgpu_peer_atomics.argtypes = [ctypes.c_int32, ctypes.c_char_p]
    L.mpgpu_peer_atomics.restype = ctypes.c_int32
    L.mpgpu_plan_key_region_bytes.argtypes = [ctypes.c_void_p]
    L.mpgpu_plan_key_region_bytes.restype = ctypes.c_int64
    L.mpgpu_plan_key_region_owners.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                               ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, _dp]
    L.mpgpu_plan_key_region_owners.restype = ctypes.c_int64
    L.mpgpu_plan_attach_key_region.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.c_int32]
    L.mpgpu_plan_attach_key_region.restype = ctypes.c_int
    L.mpgpu_plan_num_bands.argtypes = [ctypes.c_void_p]
    L.mpgpu_plan_num_bands.restype = ctypes.c_int64
    L.mpgpu_simple_join.argtypes = [ctypes.POINTER(_SimpleArgs)]
    L.mpgpu_simple_join.restype = ctypes.c_int
    L.mpgpu_mstomp.argtypes = [ctypes.POINTER(_MStompArgs)]
    L.mpgpu_mstomp.restype = ctypes.c_int
    _lib = L
    return L


def _check(status: int) -> None:
    if status == MPGPU_OK:
        return
    msg = lib().mpgpu_last_error().decode(errors="replace")
    if status == MPGPU_EUNSUPPORTED:
        raise UnsupportedError(msg)
    if status == MPGPU_EPARAM:
        raise ParameterError(msg)
    raise RuntimeError(f"mprof_b200 error {status}: {msg}")


# --------------------------------------------------------------------- results
@dataclass
class MatrixProfile:
    """Mirror of mprof::MatrixProfile (profile.hpp:28-46)."""
    values: np.ndarray
    index: np.ndarray
    left_index: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    right_index: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))
    window: int = 0
    exclusion_zone: int = 0
    mode: str = "stomp"
    join_kind: str = "self"
    coverage: float = 1.0
    seed: int = 0
    data_len: int = 0
    data_len_b: int = 0
    data_dims: int = 1

    def size(self) -> int:
        return int(self.values.size)

    def full_coverage(self) -> bool:
        return self.coverage >= 1.0

    def has_left_right(self) -> bool:
        return self.left_index.size > 0


# --------------------------------------------------------------------- helpers
def _series(x, name: str) -> np.ndarray:
    """TimeSeries validation (types.cpp:7-18): length >= 4, all finite."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    if a.size < MIN_WINDOW:
        raise ParameterError(f"time series too short: length {a.size} < minimum {MIN_WINDOW}")
    bad = np.flatnonzero(~np.isfinite(a))
    if bad.size:
        raise ParameterError(f"time series sample {int(bad[0])} is not finite")
    return a


def _check_window(w: int, n: int, what: str) -> None:
    if w < MIN_WINDOW:
        raise ParameterError(f"window {w} < minimum {MIN_WINDOW}")
    if w > n:
        raise ParameterError(f"window {w} exceeds {what} length {n}")


def zone_size(window: int, fraction: float) -> int:
    """round-half-up(window * fraction) (distance.hpp:19-20)."""
    if not (fraction >= 0.0):
        raise ParameterError("exclusion-zone fraction must be >= 0")
    return int(lib().mpgpu_zone_size(int(window), float(fraction)))


def join_cells(n_a: int, n_b: int, window: int, zone: int) -> int:
    """Unique cells of a join (self-join when n_b == 0)."""
    return int(lib().mpgpu_join_cells(int(n_a), int(n_b), int(window), int(zone)))


def _ptr(a: Optional[np.ndarray], typ):
    return a.ctypes.data_as(typ) if a is not None else None


def join(a, b=None, window: int = 4, zone: int = 0, *, n_gpus: int = 1,
         devices: Optional[Sequence[int]] = None, want_b: bool = True,
         progress: Optional[Callable[[float], None]] = None, timed: bool = False,
         out: Optional[dict] = None):
    """Raw host-buffer join through ``mpgpu_join`` (zone already resolved).

    Returns a dict with mp_a, pi_a (+ left_a, right_a for self-joins; mp_b,
    pi_b for AB-joins) and, when ``timed``, kernel_ms / total_ms. ``out`` may
    supply some or all of those arrays (C-contiguous, right dtype and length),
    e.g. views of pinned host memory so the device-to-host copies run at full
    speed; missing ones are allocated.
    """
    A = _series(a, "series")
    B = _series(b, "series B") if b is not None else None
    _check_window(window, A.size, "series")
    if B is not None:
        _check_window(window, B.size, "series B")
    La = A.size - window + 1
    given = dict(out or {})

    def _buf(name, n, dtype):
        v = given.get(name)
        if v is None:
            return np.empty(n, dtype)
        if not (isinstance(v, np.ndarray) and v.dtype == dtype and v.shape == (n,)
                and v.flags.c_contiguous and v.flags.writeable):
            raise ParameterError(f"out[{name!r}] must be a writable contiguous {np.dtype(dtype)} array of length {n}")
        return v
    out = {"mp_a": _buf("mp_a", La, np.float64), "pi_a": _buf("pi_a", La, np.int64)}
    args = _JoinArgs()
    args.a = _ptr(A, _dp)
    args.n_a = A.size
    args.b = _ptr(B, _dp)
    args.n_b = 0 if B is None else B.size
    args.window = int(window)
    args.zone = int(zone) if B is None else 0
    args.n_gpus = int(n_gpus)
    dev_arr = None
    if devices is not None:
        dev_arr = (ctypes.c_int32 * len(devices))(*devices)
        args.devices = ctypes.cast(dev_arr, ctypes.POINTER(ctypes.c_int32))
        args.n_gpus = len(devices)
    args.mp_a = _ptr(out["mp_a"], _dp)
    args.pi_a = _ptr(out["pi_a"], _ip)
    if B is None:
        out["left_a"] = _buf("left_a", La, np.int64)
        out["right_a"] = _buf("right_a", La, np.int64)
        args.left_a = _ptr(out["left_a"], _ip)
        args.right_a = _ptr(out["right_a"], _ip)
    elif want_b:
        Lb = B.size - window + 1
        out["mp_b"] = _buf("mp_b", Lb, np.float64)
        out["pi_b"] = _buf("pi_b", Lb, np.int64)
        args.mp_b = _ptr(out["mp_b"], _dp)
        args.pi_b = _ptr(out["pi_b"], _ip)
    cb = None
    if progress is not None:
        cb = _PROGRESS(lambda f, _ctx: progress(f))
        args.progress = cb
    if timed:
        k = ctypes.c_double(0)
        t = ctypes.c_double(0)
        _check(lib().mpgpu_join_timed(ctypes.byref(args), ctypes.byref(k), ctypes.byref(t)))
        out["kernel_ms"], out["total_ms"] = k.value, t.value
    else:
        _check(lib().mpgpu_join(ctypes.byref(args)))
    del dev_arr, cb
    return out


def stomp(ts_a, ts_b=None, window: int = 4, ez_fraction: float = 0.5, n_workers: int = 1,
          progress: Optional[Callable[[float], None]] = None, *, n_gpus: int = 1,
          devices: Optional[Sequence[int]] = None) -> MatrixProfile:
    """mprof::stomp (profile.hpp:80-83) on the B200. ts_b None -> self-join."""
    if n_workers < 1:
        raise ParameterError("n_workers must be >= 1")
    A = _series(ts_a, "series")
    B = _series(ts_b, "series B") if ts_b is not None else None
    _check_window(window, A.size, "series")
    if B is not None:
        _check_window(window, B.size, "series B")
    zone = zone_size(window, ez_fraction)
    r = join(A, B, window, zone, n_gpus=n_gpus, devices=devices, want_b=False, progress=progress)
    mp = MatrixProfile(values=r["mp_a"], index=r["pi_a"], window=window, mode="stomp",
                       data_len=A.size)
    if B is None:
        mp.left_index, mp.right_index = r["left_a"], r["right_a"]
        mp.exclusion_zone = zone
    else:
        mp.join_kind = "ab"
        mp.data_len_b = B.size
    return mp


def stomp_ab(ts_a, ts_b, window: int, *, n_gpus: int = 1):
    """Both AB-join profiles from one pass: (A against B, B against A)."""
    A, B = _series(ts_a, "series"), _series(ts_b, "series B")
    _check_window(window, A.size, "series")
    _check_window(window, B.size, "series B")
    r = join(A, B, window, 0, n_gpus=n_gpus, want_b=True)
    pa = MatrixProfile(values=r["mp_a"], index=r["pi_a"], window=window, join_kind="ab",
                       data_len=A.size, data_len_b=B.size)
    pb = MatrixProfile(values=r["mp_b"], index=r["pi_b"], window=window, join_kind="ab",
                       data_len=B.size, data_len_b=A.size)
    return pa, pb


BAND = 256  # diagonals per band (kW): the granularity of anytime SCRIMP subsets


def scrimp_bands(n: int, window: int, zone: int, s_size: int, seed: int = 0):
    """Band ids (ascending) and coverage of the anytime subset mpgpu_scrimp runs.

    Band b holds diagonals [zone+1 + 256 b, zone+1 + 256 (b+1)), cut at L."""
    L = n - window + 1
    nb = max(0, -(-(L - zone - 1) // BAND))
    out = np.empty(max(nb, 1), np.int64)
    cov = ctypes.c_double(0)
    k = lib().mpgpu_scrimp_bands(int(n), int(window), int(zone), int(s_size), ctypes.c_uint64(seed),
                                 out.ctypes.data_as(_ip), out.size, ctypes.byref(cov))
    return out[:k].copy(), cov.value


def scrimp_diagonals(n: int, window: int, zone: int, s_size: int, seed: int = 0):
    """(diagonals ascending, coverage) that scrimp(granularity="diagonal") evaluates."""
    L = n - window + 1
    cap = max(1, L - zone - 1)
    out = np.empty(cap, dtype=np.int64)
    cov = ctypes.c_double(0)
    k = lib().mpgpu_scrimp_diagonals(n, window, zone, s_size, ctypes.c_uint64(seed), _ptr(out, _ip), cap,
                                     ctypes.byref(cov))
    return out[:k].copy(), cov.value


def band_diagonals(bands, L: int, zone: int) -> np.ndarray:
    """Explicit diagonal list of a band subset."""
    parts = [np.arange(zone + 1 + b * BAND, min(zone + 1 + (b + 1) * BAND, L)) for b in bands]
    return np.concatenate(parts) if parts else np.empty(0, np.int64)


def scrimp(ts_a, window: int = 4, ez_fraction: float = 0.5, s_size: int = K_FULL_RUN,
           seed: int = 0, progress: Optional[Callable[[float], None]] = None,
           ts_b=None, granularity: str = "diagonal") -> MatrixProfile:
    """mprof::scrimp (profile.hpp:85-89): self-join with the anytime property.

    granularity="diagonal" (the reference's semantics): exactly s_size
    diagonals in SCRIMP's seeded order (scrimp_diagonals), coverage =
    s_size / all diagonals. granularity="band": the fast path, whole
    256-diagonal bands in a seeded order until s_size diagonals are covered.
    At full coverage the result is the exact join with left/right indexes;
    below it values are exact minima over the computed diagonals and
    left/right are absent. AB-joins raise
    UnsupportedError."""
    if granularity not in ("diagonal", "band"):
        raise ParameterError("granularity must be 'diagonal' or 'band'")
    if ts_b is not None:
        raise UnsupportedError("SCRIMP supports self-joins only")
    if s_size < 1:
        raise ParameterError("s_size must be >= 1")
    A = _series(ts_a, "series")
    _check_window(window, A.size, "series")
    zone = zone_size(window, ez_fraction)
    L = A.size - window + 1
    n_diag = max(0, L - zone - 1)
    if s_size >= n_diag:
        r = join(A, None, window, zone, progress=progress)
        return MatrixProfile(values=r["mp_a"], index=r["pi_a"], left_index=r["left_a"],
                             right_index=r["right_a"], window=window, exclusion_zone=zone,
                             mode="scrimp", seed=seed, data_len=A.size)
    mp_a = np.empty(L)
    pi_a = np.empty(L, np.int64)
    left = np.empty(L, np.int64)
    right = np.empty(L, np.int64)
    args = _JoinArgs()
    args.a = _ptr(A, _dp)
    args.n_a = A.size
    args.window = int(window)
    args.zone = zone
    args.n_gpus = 1
    args.mp_a, args.pi_a = _ptr(mp_a, _dp), _ptr(pi_a, _ip)
    args.left_a, args.right_a = _ptr(left, _ip), _ptr(right, _ip)
    cov = ctypes.c_double(0)
    fn = lib().mpgpu_scrimp if granularity == "diagonal" else lib().mpgpu_scrimp_banded
    _check(fn(ctypes.byref(args), int(s_size), ctypes.c_uint64(seed), ctypes.byref(cov)))
    full = cov.value >= 1.0
    return MatrixProfile(values=mp_a, index=pi_a,
                         left_index=left if full else np.empty(0, np.int64),
                         right_index=right if full else np.empty(0, np.int64),
                         window=window, exclusion_zone=zone, mode="scrimp", coverage=cov.value,
                         seed=seed, data_len=A.size)


# --------------------------------------------------------------- device plans
class _CudaArray:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, n: int, typestr: str, owner):
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3, "strides": None,
        }
        self._owner = owner


def _dev_ptr(t) -> int:
    if t is None:
        return 0
    if not t.is_cuda or not t.is_contiguous():
        raise ParameterError("expected a contiguous CUDA tensor")
    return int(t.data_ptr())


class Plan:
    """Device-resident join over torch CUDA float64 tensors (mpgpu_plan_*)."""

    def __init__(self, a, b=None, window: int = 4, zone: int = 0, stream=None):
        import torch  # plumbing only: device memory and streams
        if a.dtype != torch.float64 or (b is not None and b.dtype != torch.float64):
            raise ParameterError("series must be float64")
        _check_window(window, a.numel(), "series")
        if b is not None:
            _check_window(window, b.numel(), "series B")
        self.a, self.b = a, b
        self.window = int(window)
        self.self_join = b is None
        self.zone = int(zone) if b is None else 0
        self.device = a.device.index if a.device.index is not None else torch.cuda.current_device()
        self.stream = stream if stream is not None else torch.cuda.current_stream(a.device)
        self.La = a.numel() - window + 1
        self.Lb = self.La if b is None else b.numel() - window + 1
        p = lib().mpgpu_plan_create(_dev_ptr(a), a.numel(), _dev_ptr(b) or None,
                                    0 if b is None else b.numel(), self.window, self.zone,
                                    self.device, ctypes.c_void_p(self.stream.cuda_stream))
        if not p:
            _check(MPGPU_EPARAM if b is not None or window >= MIN_WINDOW else 10)
            raise RuntimeError(lib().mpgpu_last_error().decode())
        self._p = ctypes.c_void_p(p)

    def close(self) -> None:
        p = getattr(self, "_p", None)
        if p and _lib is not None:
            try:
                _lib.mpgpu_plan_destroy(p)
            except Exception:  # interpreter shutdown
                pass
        self._p = None

    __del__ = close

    def prepare(self) -> None:
        """Stats, key reset and warm start (including the coarse join) on this GPU."""
        _check(lib().mpgpu_plan_prepare(self._p))

    def prepare_shard(self, shard: int, n_shards: int) -> None:
        """Phase 1 of a sharded prepare: this rank's shard of the coarse join.
        Min-reduce coarse_keys() across ranks, then call prepare_finish()."""
        _check(lib().mpgpu_plan_prepare_shard(self._p, int(shard), int(n_shards)))

    def prepare_finish(self) -> None:
        _check(lib().mpgpu_plan_prepare_finish(self._p))

    def coarse_keys(self):
        """(row_keys, col_keys) of the pending coarse join as int64 CUDA tensors,
        or None when the plan has no coarse phase."""
        import torch
        pr, pc = ctypes.c_void_p(), ctypes.c_void_p()
        lr, lc = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().mpgpu_plan_coarse_keys(self._p, ctypes.byref(pr), ctypes.byref(lr),
                                            ctypes.byref(pc), ctypes.byref(lc)))
        if not pr.value:
            return None
        dev = torch.device("cuda", self.device)
        r = torch.as_tensor(_CudaArray(pr.value, lr.value, "<i8", self), device=dev)
        c = torch.as_tensor(_CudaArray(pc.value, lc.value, "<i8", self), device=dev)
        return r, c

    def run(self, shard: int = 0, n_shards: int = 1) -> None:
        _check(lib().mpgpu_plan_run(self._p, int(shard), int(n_shards)))

    def cells(self, shard: int = 0, n_shards: int = 1) -> int:
        return int(lib().mpgpu_plan_shard_cells(self._p, int(shard), int(n_shards)))

    def launches(self) -> int:
        return int(lib().mpgpu_plan_launch_count(self._p))

    def attach_keys(self, row_keys=None, col_keys=None) -> None:
        """Evaluate into another plan's keys (e.g. a peer GPU's, over NVLink):
        candidates are RED.MIN'd straight into them (mpgpu_plan_attach_keys)."""
        _check(lib().mpgpu_plan_attach_keys(self._p, _dev_ptr(row_keys) or None,
                                            _dev_ptr(col_keys) or None))

    def prepare_shared(self, shard: int, n_shards: int) -> None:
        """Shared-key warm start, phase 1: stats and this shard's coarse join."""
        _check(lib().mpgpu_plan_prepare_shared(self._p, int(shard), int(n_shards)))

    def seed_shared(self, shard: int, n_shards: int) -> None:
        """Phase 2 (after the coarse keys are MIN-merged): this shard's warm-start
        cells, RED.MIN'd into the (shared) keys."""
        _check(lib().mpgpu_plan_seed_shared(self._p, int(shard), int(n_shards)))

    def coarse_key_ptrs(self):
        """(row_ptr, col_ptr) of the nested coarse plan's own keys, or (None, None)
        without a coarse phase; marks the coarse keys as shared (see coarse_run)."""
        pr, pc = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().mpgpu_plan_coarse_key_ptrs(self._p, ctypes.byref(pr), ctypes.byref(pc)))
        return pr.value, pc.value

    def attach_coarse_key_ptrs(self, row_ptr: int, col_ptr: int) -> None:
        _check(lib().mpgpu_plan_attach_coarse_keys(self._p, ctypes.c_void_p(row_ptr or None),
                                                   ctypes.c_void_p(col_ptr or None)))

    def coarse_run(self, shard: int, n_shards: int) -> None:
        """This shard of the coarse join into shared coarse keys."""
        _check(lib().mpgpu_plan_coarse_run(self._p, int(shard), int(n_shards)))

    def reset_keys(self) -> None:
        """Empty the plan's own keys (the owner, before a shared-key join)."""
        _check(lib().mpgpu_plan_reset_keys(self._p))

    def attach_key_ptrs(self, row_ptr: int, col_ptr: int) -> None:
        """attach_keys() with raw device pointers (e.g. opened from another
        process's CUDA IPC handles); 0, 0 detaches."""
        _check(lib().mpgpu_plan_attach_keys(self._p, ctypes.c_void_p(row_ptr or None),
                                            ctypes.c_void_p(col_ptr or None)))

    def key_region_bytes(self) -> int:
        """Bytes of a shared key region for this plan (fine + coarse keys)."""
        return int(lib().mpgpu_plan_key_region_bytes(self._p))

    def attach_key_region(self, base: int, nbytes: int, owner: bool) -> None:
        """Keep this plan's keys (and coarse keys) in a shared region, e.g. a
        striped one (distributed.SharedKeys); base 0 detaches."""
        _check(lib().mpgpu_plan_attach_key_region(self._p, ctypes.c_void_p(base or None),
                                                  int(nbytes), 1 if owner else 0))

    def key_region_owners(self, chunk_bytes: int, n_ranks: int):
        """(owners, max_share): chunk owners of a striped key region balancing the
        modelled key reads per GPU, and the busiest rank's share of them."""
        n = int(lib().mpgpu_plan_key_region_owners(self._p, int(chunk_bytes), int(n_ranks), None, 0, None))
        if n < 0:
            raise ParameterError("bad chunk size or rank count")
        own = (ctypes.c_int32 * max(n, 1))()
        share = ctypes.c_double()
        lib().mpgpu_plan_key_region_owners(self._p, int(chunk_bytes), int(n_ranks), own, n,
                                           ctypes.byref(share))
        return list(own)[:n], share.value

    def key_ptrs(self):
        """(row_ptr, col_ptr): device addresses of the plan's own key arrays."""
        pr, pc = ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib().mpgpu_plan_keys(self._p, ctypes.byref(pr), None, ctypes.byref(pc), None))
        return pr.value, pc.value

    def keys(self):
        """(row_keys, col_keys) as int64 CUDA tensors aliasing the plan's keys."""
        import torch
        pr, pc = ctypes.c_void_p(), ctypes.c_void_p()
        lr, lc = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().mpgpu_plan_keys(self._p, ctypes.byref(pr), ctypes.byref(lr), ctypes.byref(pc),
                                     ctypes.byref(lc)))
        dev = torch.device("cuda", self.device)
        r = torch.as_tensor(_CudaArray(pr.value, lr.value, "<i8", self), device=dev)
        c = torch.as_tensor(_CudaArray(pc.value, lc.value, "<i8", self), device=dev)
        return r, c

    def finalize(self, mp_a=None, pi_a=None, left_a=None, right_a=None, mp_b=None, pi_b=None):
        _check(lib().mpgpu_plan_finalize(self._p, *[ctypes.c_void_p(_dev_ptr(t) or None)
                                                     for t in (mp_a, pi_a, left_a, right_a, mp_b, pi_b)]))

    def finalize_shard(self, shard: int, n_shards: int, mp_a=None, pi_a=None, left_a=None,
                       right_a=None, mp_b=None, pi_b=None):
        """Decode this shard's rows of every output (mpgpu_plan_finalize_shard)."""
        _check(lib().mpgpu_plan_finalize_shard(self._p, int(shard), int(n_shards),
                                               *[ctypes.c_void_p(_dev_ptr(t) or None)
                                                 for t in (mp_a, pi_a, left_a, right_a, mp_b, pi_b)]))

    def outputs(self):
        """Allocate and fill the MatrixProfile arrays on the device."""
        import torch
        dev = self.a.device
        o = {"mp_a": torch.empty(self.La, dtype=torch.float64, device=dev),
             "pi_a": torch.empty(self.La, dtype=torch.int64, device=dev)}
        if self.self_join:
            o["left_a"] = torch.empty(self.La, dtype=torch.int64, device=dev)
            o["right_a"] = torch.empty(self.La, dtype=torch.int64, device=dev)
        else:
            o["mp_b"] = torch.empty(self.Lb, dtype=torch.float64, device=dev)
            o["pi_b"] = torch.empty(self.Lb, dtype=torch.int64, device=dev)
        self.finalize(o["mp_a"], o["pi_a"], o.get("left_a"), o.get("right_a"), o.get("mp_b"),
                      o.get("pi_b"))
        return o


def distance_profiles(ts, window: int, queries=None, positions=None, zone: int = -1, stream=None,
                      out=None):
    """MASS distance-profile batch on the GPU (mass_distance_profile, distance.hpp:26-33).

    ts: float64 CUDA tensor. Either `queries` (Q x window float64 CUDA tensor,
    external windows) or `positions` (Q int64 CUDA tensor of window starts in
    ts; |j - pos| <= zone -> +inf, zone < 0: none). Returns a Q x L tensor,
    written into `out` when given (contiguous float64, same device)."""
    import torch
    _check_window(window, ts.numel(), "series")
    L = ts.numel() - window + 1
    if (queries is None) == (positions is None):
        raise ParameterError("pass exactly one of queries / positions")
    Q = queries.shape[0] if queries is not None else positions.numel()
    if queries is not None and (queries.dim() != 2 or queries.shape[1] != window):
        raise ParameterError("queries must be Q x window")
    if out is None:
        out = torch.empty((Q, L), dtype=torch.float64, device=ts.device)
    elif (tuple(out.shape) != (Q, L) or out.dtype != torch.float64 or out.device != ts.device
          or not out.is_contiguous()):
        raise ParameterError(f"out must be a contiguous float64 ({Q}, {L}) tensor on {ts.device}")
    st = stream if stream is not None else torch.cuda.current_stream(ts.device)
    _check(lib().mpgpu_distance_profiles(
        _dev_ptr(ts), ts.numel(), int(window),
        _dev_ptr(queries.contiguous()) if queries is not None else None,
        _dev_ptr(positions.contiguous()) if positions is not None else None,
        int(Q), int(zone), _dev_ptr(out), ts.device.index or 0, ctypes.c_void_p(st.cuda_stream)))
    return out


def mass_distance_profile(query, ts, query_index: int = -1, ez_zone: int = 0) -> np.ndarray:
    """Host mirror of mprof::mass_distance_profile (distance.hpp:30-33) on the GPU."""
    import torch
    q = _series(query, "query")
    t = _series(ts, "series")
    _check_window(q.size, t.size, "series")
    d = torch.from_numpy(t).cuda()
    if query_index >= 0:
        out = distance_profiles(d, q.size, positions=torch.tensor([query_index], device=d.device),
                                zone=ez_zone)
    else:
        out = distance_profiles(d, q.size, queries=torch.from_numpy(q).cuda().view(1, -1))
    return out[0].cpu().numpy()


def _extract(d_values, k, zone, largest, stop_at):
    import torch
    idx = np.empty(max(int(k), 1), np.int64)
    val = np.empty(max(int(k), 1))
    st = torch.cuda.current_stream(d_values.device)
    got = lib().mpgpu_extract(_dev_ptr(d_values), d_values.numel(), int(k), int(zone), int(largest),
                              float(stop_at), idx.ctypes.data_as(_ip), val.ctypes.data_as(_dp),
                              d_values.device.index or 0, ctypes.c_void_p(st.cuda_stream))
    if got < 0:
        _check(MPGPU_EPARAM)
    return idx[:got].copy(), val[:got].copy()


def find_discord(profile: MatrixProfile, n_discords: int, zone: int = -1):
    """find_discord (discovery.hpp:61-63) on the GPU: repeated argmax of the
    finite profile values, masking +-zone around each hit (zone < 0: the
    profile's own exclusion zone). Returns (list of (index, distance), truncated)."""
    import torch
    if n_discords < 0:
        raise ParameterError("n_discords must be >= 0")
    z = profile.exclusion_zone if zone < 0 else int(zone)
    d = torch.from_numpy(np.ascontiguousarray(profile.values, dtype=np.float64)).cuda()
    idx, val = _extract(d, n_discords, z, True, -np.inf)
    return list(zip(idx.tolist(), val.tolist())), bool(idx.size < n_discords)


def fluss(profile_index, window: int):
    """fluss_arc_count + fluss_cac (discovery.hpp:68-74) on the GPU.
    Returns (arc_counts int64, cac float64) as numpy arrays."""
    import torch
    ix = torch.from_numpy(np.ascontiguousarray(profile_index, dtype=np.int64)).cuda()
    L = ix.numel()
    arcs = torch.empty(L, dtype=torch.int64, device=ix.device)
    cac = torch.empty(L, dtype=torch.float64, device=ix.device)
    st = torch.cuda.current_stream(ix.device)
    _check(lib().mpgpu_fluss(_dev_ptr(ix), L, int(window), _dev_ptr(arcs), _dev_ptr(cac),
                             ix.device.index or 0, ctypes.c_void_p(st.cuda_stream)))
    return arcs.cpu().numpy(), cac.cpu().numpy()


def fluss_extract(cac, num_segments: int, window: int, exclusion_factor: float = 5.0):
    """fluss_extract (discovery.hpp:76-79): repeated argmin over the CAC, masking
    +-exclusion_factor*window, stopping once nothing below 1 remains.
    Returns (segment positions, truncated)."""
    import torch
    c = torch.from_numpy(np.ascontiguousarray(cac, dtype=np.float64)).cuda()
    zone = int(np.floor(exclusion_factor * window))
    idx, _ = _extract(c, num_segments, zone, False, 1.0)
    return idx.tolist(), bool(idx.size < num_segments)


def rolling_stats(ts, window: int, stream=None):
    """rolling_mean_std (rolling.hpp:25-29) of a float64 CUDA tensor."""
    import torch
    _check_window(window, ts.numel(), "series")
    L = ts.numel() - window + 1
    mu = torch.empty(L, dtype=torch.float64, device=ts.device)
    sd = torch.empty(L, dtype=torch.float64, device=ts.device)
    st = stream if stream is not None else torch.cuda.current_stream(ts.device)
    _check(lib().mpgpu_rolling_stats(_dev_ptr(ts), ts.numel(), int(window), _dev_ptr(mu),
                                     _dev_ptr(sd), ts.device.index or 0,
                                     ctypes.c_void_p(st.cuda_stream)))
    return mu, sd


# ----------------------------------------------------------------- multivariate
class MultiTimeSeries:
    """Mirror of mprof::MultiTimeSeries (types.hpp:43-53; ctor types.cpp:20-32):
    d >= 1 dimensions of equal length, each a validated TimeSeries. Built from
    a (d, n) array or a sequence of 1-D series; ``data`` is dim-major."""

    def __init__(self, dims):
        if isinstance(dims, MultiTimeSeries):
            self.data = dims.data
            return
        if isinstance(dims, np.ndarray) and dims.ndim == 2:
            rows = [dims[q] for q in range(dims.shape[0])]
        elif isinstance(dims, np.ndarray) and dims.ndim == 1:
            rows = [dims]
        else:
            rows = list(dims)
        if not rows:
            raise ParameterError("multivariate series needs at least one dimension")
        rows = [_series(r, f"dimension {q}") for q, r in enumerate(rows)]
        n = rows[0].size
        for q, r in enumerate(rows[1:], 1):
            if r.size != n:
                raise ParameterError(f"dimension {q} has length {r.size}, expected {n}")
        self.data = np.ascontiguousarray(np.stack(rows))

    def dims(self) -> int:
        return int(self.data.shape[0])

    def size(self) -> int:
        return int(self.data.shape[1])

    def dim(self, k: int) -> np.ndarray:
        return self.data[k]


@dataclass
class MultiMatrixProfile:
    """Mirror of mprof::MultiMatrixProfile (profile.hpp:48-62): row k is the
    best (k+1)-dimensional profile; dim_order[k][i] the dimension filling slot
    k at the chosen partner (-1 for an exhausted selection)."""
    values: np.ndarray
    index: np.ndarray
    dim_order: np.ndarray
    window: int = 0
    exclusion_zone: int = 0
    must_dims: tuple = ()
    exc_dims: tuple = ()
    data_len: int = 0
    data_dims: int = 0

    def size(self) -> int:
        return 0 if self.values.size == 0 else int(self.values.shape[1])


def simple_join(mts_a, mts_b=None, window: int = 4, ez_fraction: float = 0.5,
                progress: Optional[Callable[[float], None]] = None, *, device: int = 0,
                want_b: bool = False, timed: bool = False):
    """mprof::simple_join (profile.hpp:96-100): SiMPle on the B200.

    Non-normalised Euclidean distance summed over all dimensions; mts_b None
    -> self-join (exclusion zone, left / right filled), else AB-join (zone 0).
    ``want_b`` also returns B's profile against A from the same pass (as a
    second MatrixProfile); ``timed`` attaches ``kernel_ms``."""
    A = MultiTimeSeries(mts_a)
    B = MultiTimeSeries(mts_b) if mts_b is not None else None
    if B is not None and B.dims() != A.dims():
        raise ParameterError(f"dimension mismatch: {A.dims()} vs {B.dims()}")
    _check_window(window, A.size(), "series")
    if B is not None:
        _check_window(window, B.size(), "series B")
    zone = zone_size(window, ez_fraction) if B is None else 0
    La = A.size() - window + 1
    mp_a, pi_a = np.empty(La), np.empty(La, np.int64)
    args = _SimpleArgs()
    args.a = _ptr(A.data, _dp)
    args.n_a = A.size()
    args.b = _ptr(B.data, _dp) if B is not None else None
    args.n_b = 0 if B is None else B.size()
    args.dims = A.dims()
    args.window = int(window)
    args.zone = int(zone)
    args.device = int(device)
    args.mp_a = _ptr(mp_a, _dp)
    args.pi_a = _ptr(pi_a, _ip)
    left = right = mp_b = pi_b = None
    if B is None:
        left, right = np.empty(La, np.int64), np.empty(La, np.int64)
        args.left_a, args.right_a = _ptr(left, _ip), _ptr(right, _ip)
    elif want_b:
        Lb = B.size() - window + 1
        mp_b, pi_b = np.empty(Lb), np.empty(Lb, np.int64)
        args.mp_b, args.pi_b = _ptr(mp_b, _dp), _ptr(pi_b, _ip)
    kms = ctypes.c_double(0)
    args.kernel_ms = ctypes.pointer(kms)
    _check(lib().mpgpu_simple_join(ctypes.byref(args)))
    if progress is not None:
        progress(1.0)
    prof = MatrixProfile(values=mp_a, index=pi_a, window=window, mode="simple",
                         data_len=A.size(), data_dims=A.dims())
    if B is None:
        prof.left_index, prof.right_index = left, right
        prof.exclusion_zone = zone
    else:
        prof.join_kind = "ab"
        prof.data_len_b = B.size()
    if timed:
        prof.kernel_ms = kms.value
    if want_b and B is not None:
        pb = MatrixProfile(values=mp_b, index=pi_b, window=window, mode="simple", join_kind="ab",
                           data_len=B.size(), data_len_b=A.size(), data_dims=A.dims())
        return prof, pb
    return prof


def mstomp(mts, window: int = 4, ez_fraction: float = 0.5, must_dims: Sequence[int] = (),
           exc_dims: Sequence[int] = (), n_workers: int = 1,
           progress: Optional[Callable[[float], None]] = None, *, device: int = 0,
           timed: bool = False) -> MultiMatrixProfile:
    """mprof::mstomp (profile.hpp:91-94): k-dimensional profiles for every k,
    self-join only. Errors: must / exc overlap, repeated or
    out-of-range dims, or every dim excluded -> ParameterError."""
    if n_workers < 1:
        raise ParameterError("n_workers must be >= 1")
    X = MultiTimeSeries(mts)
    _check_window(window, X.size(), "series")
    zone = zone_size(window, ez_fraction)
    d, L = X.dims(), X.size() - window + 1
    must = np.ascontiguousarray(list(must_dims), dtype=np.int64)
    exc = np.ascontiguousarray(list(exc_dims), dtype=np.int64)
    vals = np.empty((d, L))
    idx = np.empty((d, L), np.int64)
    dorder = np.empty((d, L), np.int64)
    args = _MStompArgs()
    args.x = _ptr(X.data, _dp)
    args.n = X.size()
    args.dims = d
    args.window = int(window)
    args.zone = int(zone)
    args.must_dims = _ptr(must, _ip) if must.size else None
    args.n_must = must.size
    args.exc_dims = _ptr(exc, _ip) if exc.size else None
    args.n_exc = exc.size
    args.device = int(device)
    args.mp = _ptr(vals, _dp)
    args.pi = _ptr(idx, _ip)
    args.dim_order = _ptr(dorder, _ip)
    kms = ctypes.c_double(0)
    args.kernel_ms = ctypes.pointer(kms)
    _check(lib().mpgpu_mstomp(ctypes.byref(args)))
    if progress is not None:
        progress(1.0)
    r = MultiMatrixProfile(values=vals, index=idx, dim_order=dorder, window=window,
                           exclusion_zone=zone, must_dims=tuple(int(q) for q in must),
                           exc_dims=tuple(int(q) for q in exc), data_len=X.size(), data_dims=d)
    if timed:
        r.kernel_ms = kms.value
    return r
