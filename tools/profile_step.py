#!/usr/bin/env python3
"""One join step (stats + k_join + finalize) of a config, for ncu captures.

    python tools/profile_step.py --config C4 [--steps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1904_12626_b200 as mp  # noqa: E402
from paper_1904_12626_b200 import datasets  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--n", type=int, default=0, help="override series length (self-joins)")
args = ap.parse_args()
kw = {"n": args.n} if args.n else {}
cfg = datasets.get(args.config, **kw)
a = torch.from_numpy(cfg.a).cuda()
b = torch.from_numpy(cfg.b).cuda() if cfg.b is not None else None
plan = mp.Plan(a, b, cfg.window, cfg.zone)
for _ in range(args.steps):
    plan.prepare()
    plan.run(0, 1)
    o = plan.outputs()
torch.cuda.synchronize()
print({"config": cfg.name, "cells": plan.cells(), "launches_per_step": plan.launches(),
       "mp_min": float(o["mp_a"].min()), "mp_max": float(o["mp_a"][torch.isfinite(o["mp_a"])].max())})
