"""One sort of a BASELINE config for ncu captures (no warm-up, deterministic
kernel order: the first launch of each kernel is the root level).

    python profiles/profile_one.py --config 2 [--n N] [--cfg key=value ...]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--cfg", action="append", default=[])
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_1305_1157_b200 import datasets
    from paper_1305_1157_b200.samplesort import SampleSortConfig, gpu_sort
    kw = {}
    for item in a.cfg:
        k, _, v = item.partition("=")
        kw[k] = int(v) if v.lstrip("-").isdigit() else v
    cfg = SampleSortConfig(**kw)
    arena, h0 = datasets.generate(a.config, a.n)
    d0 = torch.from_numpy(h0).cuda()
    lcp = torch.empty(h0.size - 1, dtype=torch.int64, device="cuda")
    for _ in range(a.reps):
        d = d0.clone()
        gpu_sort(arena, d, 0, cfg, lcp)
    torch.cuda.synchronize()
    print("ok", h0.size)


if __name__ == "__main__":
    main()
