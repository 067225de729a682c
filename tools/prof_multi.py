"""One multivariate join for ncu: python tools/prof_multi.py simple|mstomp dims n window."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_12626_b200 as mp  # noqa: E402

kind, d, n, w = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
x = np.cumsum(np.random.default_rng(2018).standard_normal((d, n)), axis=1)
r = (mp.simple_join(x, None, w, 0.5, timed=True) if kind == "simple" else mp.mstomp(x, w, 0.5, timed=True))
print(kind, d, n, w, "kernel_ms", r.kernel_ms)
