"""The C-ABI library and the host-side API without a GPU.

Checks that libmprof_b200.so loads and exports every entry point
include/mprof_gpu.h declares, that the CPU-only entry points answer, that
parameter errors come back as the reference's error types before any device
work, and that the drop-in C++ headers compile.
"""
import ctypes
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mp():
    import paper_1904_12626_b200 as mp
    from paper_1904_12626_b200 import build
    build.build()  # no-op when up to date
    mp.lib()
    return mp


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mprof_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(mpgpu_[a-z_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol(mp):
    lib = ctypes.CDLL(mp._LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1904_12626_b200", "libmprof_b200.so")
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump absent")
    out = subprocess.run([cuobjdump, "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_cpu_entry_points(mp):
    assert mp.zone_size(50, 0.5) == 25 and mp.zone_size(80, 0.5) == 40 and mp.zone_size(50, 0.25) == 13
    with pytest.raises(mp.ParameterError):
        mp.zone_size(10, -1.0)
    # unique-cell counts
    assert mp.join_cells(16384, 0, 256, 128) == (16129 - 128 - 1) * (16129 - 128) // 2
    assert mp.join_cells(262144, 65536, 512, 0) == 261633 * 65025
    assert mp.join_cells(10, 0, 10, 5) == 0
    info = mp.lib().mpgpu_build_info().decode()
    assert "sm_100a" in info and "fp64" in info


def test_parameter_errors_before_device_work(mp):
    x = np.cumsum(np.random.default_rng(0).standard_normal(100))
    with pytest.raises(mp.ParameterError):
        mp.stomp(x[:3], None, 4)                    # series shorter than kMinWindow
    with pytest.raises(mp.ParameterError):
        mp.stomp(np.r_[x, np.nan], None, 8)         # non-finite sample
    with pytest.raises(mp.ParameterError):
        mp.stomp(x, None, 3)                        # window below minimum
    with pytest.raises(mp.ParameterError):
        mp.stomp(x, None, 101)                      # window longer than series
    with pytest.raises(mp.ParameterError):
        mp.stomp(x, x[:10], 20)                     # AB: B shorter than window
    with pytest.raises(mp.ParameterError):
        mp.stomp(x, None, 10, -0.5)                 # negative zone fraction
    with pytest.raises(mp.UnsupportedError):
        mp.scrimp(x, 10, 0.5, ts_b=x)               # AB-join SCRIMP
    with pytest.raises(mp.ParameterError):
        mp.scrimp(x, 10, 0.5, s_size=0)             # s_size < 1
    assert issubclass(mp.UnsupportedError, mp.ParameterError)
    # the C ABI itself rejects bad windows with MPGPU_EPARAM (no device touched)
    args = mp._JoinArgs()
    a = np.ascontiguousarray(x)
    args.a = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    args.n_a = a.size
    args.window = 3
    assert mp.lib().mpgpu_join(ctypes.byref(args)) == mp.MPGPU_EPARAM
    assert b"window" in mp.lib().mpgpu_last_error()
    p = mp.lib().mpgpu_plan_create(None, 100, None, 0, 8, 4, 0, None)
    assert not p


def test_anytime_band_selection_host_logic(mp):
    n, w = 100000, 256
    zone = mp.zone_size(w, 0.5)
    L = n - w + 1
    nd = L - zone - 1
    b5, c5 = mp.scrimp_bands(n, w, zone, nd // 20, 7)
    b20, c20 = mp.scrimp_bands(n, w, zone, nd // 5, 7)
    assert np.all(np.diff(b5) > 0) and set(b5) <= set(b20)     # same seed: nested subsets
    assert c5 < c20 < 1.0
    diags = mp.band_diagonals(b20, L, zone)
    assert abs(diags.size / nd - c20) < 1e-12 and diags.size >= nd // 5
    ball, call = mp.scrimp_bands(n, w, zone, 0, 7)
    assert call == 1.0 and ball.size == -(-nd // 256)
    b5b, _ = mp.scrimp_bands(n, w, zone, nd // 20, 8)
    assert not np.array_equal(b5, b5b)                          # the seed matters


def test_key_format_mirror():
    from paper_1904_12626_b200 import keys
    b = keys.index_bits(1048321)
    assert b == 20
    c = np.array([0.999, 0.5, -0.3, 1.0 + 1e-16])
    k = keys.pack(c, np.array([5, 6, 7, 8]), b)
    s, i = keys.unpack(k, b)
    assert np.array_equal(i, [5, 6, 7, 8])
    assert np.all(np.abs(s - np.maximum(1 - c, 0)) <= np.maximum(1 - c, 0) * 2.0 ** -31)
    # ordering: smaller score first, then smaller index on equal scores
    k2 = keys.pack(np.array([0.9, 0.9, 0.95]), np.array([9, 3, 12]), b)
    assert np.argmin(k2) == 2 and k2[1] < k2[0]
    assert keys.unpack(np.array([keys.KEY_NONE]), b)[1][0] == -1


def test_cpp_headers_compile():
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ absent")
    src = os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp")
    r = subprocess.run([gxx, "-std=c++20", "-fsyntax-only", "-I" + os.path.join(ROOT, "include"), src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_multivariate_parameter_errors_without_gpu(mp):
    """mpgpu_mstomp / mpgpu_simple_join reject bad arguments (SPEC.md:229,
    :240) before any device work, as the reference's ParameterError."""
    x = np.random.default_rng(1).standard_normal((3, 64))
    for must, exc in (((0,), (0,)), ((), (0, 1, 2)), ((3,), ()), ((0, 0), ()), ((), (-1,))):
        with pytest.raises(mp.ParameterError):
            mp.mstomp(x, 8, 0.5, must, exc)
    with pytest.raises(mp.ParameterError):
        mp.simple_join(x, x[:2], 8)
    with pytest.raises(mp.ParameterError):
        mp.mstomp(x, 65, 0.5)
    with pytest.raises(mp.ParameterError):
        mp.MultiTimeSeries([x[0], x[1][:50]])
    with pytest.raises(mp.ParameterError):
        mp.MultiTimeSeries([])
