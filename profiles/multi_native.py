"""Wall time of s5_sort_multi (the C-ABI multi-GPU entry) on one GPU.

    python profiles/multi_native.py [config] [n]

G = 1 shows the fixed cost around one local sort; G = 2, 4, 8 over a repeated
device list serialise their slices on the one device, so their numbers are
an upper bound of the host-side choreography (samples, splitters, partition,
peer copies), not multi-GPU throughput.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1305_1157_b200 import datasets, sort_with_lcp
from paper_1305_1157_b200.multi import sort_multi_device

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
arena, h0 = datasets.generate(cfg, n)
dev = torch.device("cuda", 0)
arena.device(dev)
out = {"config": cfg, "n": int(h0.size)}
base = torch.from_numpy(h0).to(dev)
for _ in range(3):
    h = base.clone()
    torch.cuda.synchronize()
    t = time.perf_counter()
    sort_with_lcp(arena, h)
    torch.cuda.synchronize()
    out["s5_sort_ms"] = round((time.perf_counter() - t) * 1e3, 3)
for G in (1, 2, 4, 8):
    bounds = [(h0.size * g // G, h0.size * (g + 1) // G) for g in range(G)]
    shards = [base[a:b].clone() for a, b in bounds]
    best = None
    for _ in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        slices, lcps = sort_multi_device(arena, shards, [0] * G)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        best = ms if best is None else min(best, ms)
    out[f"s5_sort_multi_G{G}_ms"] = round(best, 3)
    out[f"slices_G{G}"] = [int(s.numel()) for s in slices]
print(json.dumps(out))
