"""Build libmprof_b200.so in-tree (nvcc, sm_100a) — no JIT cache, no pip install."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmprof_b200.so")
SOURCES = ["mpgpu.cu", "mpgpu_multi.cu", "mpgpu_stripes.cpp", "mprof_api.cpp", "mprof_archive.cpp"]
HEADERS = ["mpgpu_kernels.cuh", "mpgpu_internal.h"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps():
    inc = os.path.join(ROOT, "include")
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(inc, "mprof_gpu.h")]
    deps += sorted(os.path.join(inc, "mprof", f) for f in os.listdir(os.path.join(inc, "mprof")))
    deps += [os.path.abspath(__file__)]  # the nvcc command line lives here
    return deps


def source_hash() -> str:
    """SHA-256 over the tracked sources the library is built from."""
    import hashlib
    h = hashlib.sha256()
    for d in _deps():
        h.update(os.path.relpath(d, ROOT).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


STAMP = OUT + ".stamp"


def needs_build() -> bool:
    """Rebuild unless the .so exists AND its stamp records the hash of exactly
    the current sources (an untracked or stale binary is never reused)."""
    if not os.path.exists(OUT) or not os.path.exists(STAMP):
        return True
    try:
        with open(STAMP) as f:
            return f.read().strip() != source_hash()
    except OSError:
        return True


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    cmd = [
        _nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
        "-std=c++20", "-Xcompiler", "-fPIC,-O3", "-shared", "-Xptxas", "-v",
        "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
        *[os.path.join(CSRC, s) for s in SOURCES], "-o", OUT + ".tmp",
    ]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libmprof_b200.so")
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(r.stderr)
    os.replace(OUT + ".tmp", OUT)
    with open(STAMP, "w") as f:
        f.write(source_hash() + "\n")
    if verbose:
        print(r.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
