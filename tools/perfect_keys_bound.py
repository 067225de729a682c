"""Upper bound of any warm start: time k_join when the keys already hold the exact answer.

    python tools/perfect_keys_bound.py C1,C2,C3,C4
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_12626_b200 as mp
from paper_1904_12626_b200 import datasets
for name in sys.argv[1].split(","):
    c = datasets.get(name)
    a = torch.from_numpy(c.a).cuda(); b = torch.from_numpy(c.b).cuda() if c.b is not None else None
    plan = mp.Plan(a, b, c.window, c.zone)
    res = {}
    for mode in ("normal", "perfect"):
        ts = []
        for r in range(3):
            if mode == "normal" or r == 0:
                plan.prepare()
                if mode == "perfect":
                    plan.run(0, 1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); plan.run(0, 1); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[mode] = min(ts)
    print(json.dumps({"config": name, "join_ms_normal": res["normal"], "join_ms_perfect_keys": res["perfect"]}), flush=True)
    plan.close()
