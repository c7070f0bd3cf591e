"""Phase times of distributed_sample_sort on the calling ranks (torchrun).

    torchrun --nproc-per-node G profiles/dist_phases.py --config 2

Synchronises the device between phases (so phases do not overlap) and prints
rank 0's per-phase milliseconds: the overhead budget of the multi-GPU path
around the local sort."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1305_1157_b200 import datasets, distributed as D
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G, rank = dist.get_world_size(), dist.get_rank()
    arena, h0 = datasets.generate(a.config, a.n)
    n = h0.size
    shard = torch.from_numpy(np.ascontiguousarray(h0[n * rank // G:n * (rank + 1) // G])).cuda()
    be = D.GpuBackend(arena)
    D.PHASES = {}
    for r in range(a.reps + 1):
        D.PHASES.clear()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        D.distributed_sample_sort(arena, shard.clone(), backend=be)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    if rank == 0:
        print(f"G={G} total {1e3 * (t1 - t0):.3f} ms; phases (ms):",
              {k: round(v, 3) for k, v in D.PHASES.items()})
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
