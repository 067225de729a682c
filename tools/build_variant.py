#!/usr/bin/env python3
"""Build an experiment variant of libmprof_b200.so into exp_libs/<name>.so with
extra nvcc flags (e.g. -DMPGPU_EXPERIMENT_FASTONLY); select it at run time with
MPGPU_LIB=exp_libs/<name>.so. Experiments only: the product is build.py's.

    python tools/build_variant.py fastonly -DMPGPU_EXPERIMENT_FASTONLY
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1904_12626_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "exp_libs"), exist_ok=True)
out = os.path.join(ROOT, "exp_libs", name + ".so")
cmd = [b._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++20",
       "-Xcompiler", "-fPIC,-O3", "-shared", "-Xptxas", "-v", *flags,
       "-I" + os.path.join(ROOT, "include"), "-I" + b.CSRC,
       *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-o", out]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stderr)
    sys.exit(1)
lines = r.stderr.splitlines()
for i, line in enumerate(lines):
    if "Function properties for _ZN5mpgpu6k_join" in line:
        sys.stderr.write(name + ": " + " ".join(x.strip() for x in lines[i + 1:i + 3]) + "\n")
print(out)
