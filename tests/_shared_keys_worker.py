"""torchrun worker for tests/test_gpu_shared_keys.py: the ranks share one key
region striped over their GPUs (here all on cuda:0, so every chunk is local
but every rank still maps the others' chunks from file descriptors) and join
their shards into it; rank 0 checks the profile against a one-process join of
the same series (bit-identical) and prints OK."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1904_12626_b200 as mp  # noqa: E402
from paper_1904_12626_b200.distributed import SharedKeys, shared_keys_join, sharded_join  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)  # functional test: every rank on cuda:0
    dist.init_process_group("gloo")
    n, m, ab = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == "ab"
    g = np.random.default_rng(77)
    x = np.cumsum(g.standard_normal(n))
    y = np.cumsum(g.standard_normal(n // 2)) if ab else None
    a = torch.from_numpy(x).cuda()
    b = torch.from_numpy(y).cuda() if ab else None
    zone = 0 if ab else mp.zone_size(m, 0.5)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        plan = mp.Plan(a, b, m, zone, stream=stream)
        shared = SharedKeys(plan, rank, world)
        assert shared.chunks >= 1 and shared.chunk_bytes >= 1 << 21, (shared.chunks, shared.chunk_bytes)
        outs = []
        for _ in range(2):  # the second step reuses the mappings and resets the keys
            outs.append({k: v.clone() if v is not None else v for k, v in
                         (shared_keys_join(plan, rank, world, shared=shared) or {}).items()})
        shared.close()
        sep = sharded_join(plan, rank, world)  # separate keys + MIN-reduce
    torch.cuda.synchronize()
    if rank == 0:
        ref_plan = mp.Plan(a, b, m, zone)
        ref_plan.prepare()
        ref_plan.run(0, 1)
        ref = ref_plan.outputs()
        torch.cuda.synchronize()
        for o in outs + [sep]:
            for k, v in ref.items():
                assert torch.equal(o[k], v), (k, int((o[k] != v).sum()))
        print("OK", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
