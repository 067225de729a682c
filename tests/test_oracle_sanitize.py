"""The oracle (test infrastructure) under AddressSanitizer + UBSan: every
entry point on small seeded inputs and the edge cases (window == n, zone
beyond the profile, flat runs, AB with a B of one window, single-row samples)
must run without a memory or undefined-behaviour report. The GPU library has
no such run: compute-sanitizer is closed on this pool."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_oracle_under_asan_ubsan(tmp_path):
    exe = str(tmp_path / "oracle_asan")
    srcs = [os.path.join(ROOT, "oracle", f) for f in ("mprof_oracle.c", "mprof_oracle_multi.c")]
    r = subprocess.run(["gcc", "-O1", "-g", "-fopenmp", "-fsanitize=address,undefined",
                        "-fno-sanitize-recover=all", "-fno-omit-frame-pointer",
                        "-I" + os.path.join(ROOT, "oracle"), *srcs,
                        os.path.join(ROOT, "tests", "c", "oracle_sanitize_driver.c"), "-lm", "-o", exe],
                       capture_output=True, text=True)
    if r.returncode != 0 and "sanitizer" in r.stderr.lower():
        pytest.skip("sanitizer runtime unavailable: " + r.stderr[-300:])
    assert r.returncode == 0, r.stderr[-3000:]
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1", OMP_NUM_THREADS="2")
    run = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=300)
    assert run.returncode == 0, run.stdout[-2000:] + run.stderr[-4000:]
    assert "checksum" in run.stdout and "runtime error" not in run.stderr
