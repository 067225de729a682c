"""Link-level drop-in check (CPU, no GPU needed): reference-API callers
compiled against the REFERENCE's own headers (/root/reference/proj/include,
present in the build container only) link against libmprof_b200.so with no
unresolved mprof:: symbol. Covers the join entry points (dropin_example.cpp:
stomp, scrimp, mstomp, simple_join) and the path's primitives
(primitives_example.cpp: rolling_mean_std, is_flat_std, znorm_dist_from_qt,
zone_size, apply_exclusion_zone[_inplace], mass_distance_profile, merge_min).
The same callers run against the GPU in tests/test_dropin_cpp.py."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
LIB = os.path.join(ROOT, "paper_1904_12626_b200", "libmprof_b200.so")


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present (GPU box)")
@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
@pytest.mark.parametrize("src", ["dropin_example.cpp", "primitives_example.cpp"])
def test_reference_headers_link(src, tmp_path):
    gxx = shutil.which("g++")
    libdir = os.path.dirname(LIB)
    out = str(tmp_path / "caller")
    # -Wl,--no-undefined + --unresolved-symbols=report-all: every symbol must
    # resolve at link time (libcudart comes in through the library itself)
    r = subprocess.run([gxx, "-std=c++20", "-O1", "-I" + REF_INC,
                        os.path.join(ROOT, "tests", "cpp", src), "-L" + libdir, "-lmprof_b200",
                        "-Wl,--unresolved-symbols=report-all", "-Wl,--allow-shlib-undefined",
                        "-o", out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    nm = subprocess.run(["nm", "-uC", out], capture_output=True, text=True).stdout
    need = [ln.split(None, 1)[1] for ln in nm.splitlines() if "mprof::" in ln]
    assert need, "caller uses no mprof:: symbols?"
    have = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True).stdout
    missing = [s for s in need if s not in have]
    assert not missing, missing
