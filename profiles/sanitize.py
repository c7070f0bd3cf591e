"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python profiles/sanitize.py [--quick]

Config 1 (n = 2^17 at full size, 2^14 with --quick) and the six adversarial
shapes of tests/test_gpu_parity.py (scaled down so racecheck finishes), each
under several tier configurations so every kernel runs: the wide pipeline
(both scatter variants), the narrow one-CTA step, all one-CTA local sizes, the
warp tier, k_small, k_lcp_fix; plus the host-buffer path (staging kernels),
the partition kernel, ingest, lengths and materialisation.  Every result is
checked against the oracle (test infrastructure), so a run that exits 0 is
also a parity run under the sanitizer.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (the checker)
from paper_1305_1157_b200 import (SampleSortConfig, arena_from_strings, datasets,  # noqa: E402
                                  sort_with_lcp)

CFGS = {
    "default": SampleSortConfig(),
    "wide_everywhere": SampleSortConfig(v=255, small_max=32, narrow_max=32, seed=5),
    "wide_tma": SampleSortConfig(v=255, small_max=32, narrow_max=32, seed=5, flags=32),
    "narrow_tier": SampleSortConfig(narrow_max=16384, seed=13),
    "local_small8": SampleSortConfig(v=63, small_max=8, local_max=256, narrow_max=1024),
    "tma2048": SampleSortConfig(v=255, small_max=16, narrow_max=64, flags=128),
}


def shapes(n, rng):
    yield "identical", [b"the-same-string-repeated"] * n
    yield "empty", [b""] * (n // 2) + [b"x"] * (n // 2)
    base = bytes(rng.integers(97, 123, 300).tolist())
    yield "prefix300", [base + bytes(rng.integers(97, 99, rng.integers(0, 12)).tolist())
                        for _ in range(n // 10)]
    yield "binary", [bytes(rng.integers(1, 256, rng.integers(0, 24)).tolist()) for _ in range(n)]
    yield "len1", [bytes([int(x)]) for x in rng.integers(1, 4, n)]
    yield "nested", [b"a" * int(k) for k in rng.integers(0, 120, n // 3)]


def check(name, arena, h0, cfg):
    want = h0.copy()
    O.parallel_sample_sort(arena, want, 4)
    got, lcp = sort_with_lcp(arena, h0.copy(), cfg=cfg)
    assert np.array_equal(np.sort(got), np.sort(h0)), f"{name}: not a permutation"
    assert O.contents_equal(arena, got, want), f"{name}: strings differ"
    assert np.array_equal(lcp, O.adjacent_lcps(arena, want)), f"{name}: LCP differs"
    print(f"ok {name} n={h0.size}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="smaller inputs (racecheck)")
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    n1 = 1 << (14 if a.quick else 17)
    arena, h0 = datasets.generate(1, n1)
    for cname, cfg in CFGS.items():
        check(f"config1/{cname}", arena, h0, cfg)
    for cfg_n in (2, 3, 4, 5):
        arena, h0 = datasets.generate(cfg_n, 1 << (13 if a.quick else 16))
        check(f"config{cfg_n}/default", arena, h0, CFGS["default"])
        check(f"config{cfg_n}/wide_everywhere", arena, h0, CFGS["wide_everywhere"])
    rng = np.random.default_rng(17)
    for sname, strs in shapes(20_000 if a.quick else 60_000, rng):
        arena, h0 = arena_from_strings(strs)
        for cname in ("default", "wide_everywhere", "local_small8"):
            check(f"{sname}/{cname}", arena, h0, CFGS[cname])
    # device-resident entry, partition, ingest, lengths, materialisation
    from paper_1305_1157_b200 import ingest_lines, materialize, string_lengths
    from paper_1305_1157_b200.distributed import GpuBackend
    arena, h0 = datasets.generate(1, 1 << 12)
    dev = torch.device("cuda", 0)
    d = torch.from_numpy(h0).to(dev)
    sort_with_lcp(arena, d)
    be = GpuBackend(arena)
    spl = d[torch.tensor([1000, 2000, 3000], device=dev)]
    out, counts = be.partition(torch.from_numpy(h0).to(dev), spl)
    assert sum(counts) == h0.size
    raw = b"\n".join(b"line%05d" % i for i in range(5000)) + b"\n"
    ar, hh = ingest_lines(raw)
    string_lengths(ar, hh)
    materialize(ar, hh)
    torch.cuda.synchronize()
    print("sanitize workload done", flush=True)


if __name__ == "__main__":
    main()
