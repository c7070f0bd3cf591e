"""Histogram of the segment sizes of every level of one sort (audit hook).

    python profiles/segment_sizes.py --config 3 [--n N]

Prints, per level, the number of segments and strings per size class
(<=32, <=64, <=128, <=256, <=512, <=1024, <=2048, <=4096, >4096) and their
depth range -- the shape of the recursion the local tier sees.
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=None)
    a = ap.parse_args()
    import numpy as np
    from paper_1305_1157_b200 import datasets
    from paper_1305_1157_b200._audit import audited_sort
    from paper_1305_1157_b200.samplesort import SampleSortConfig
    arena, h = datasets.generate(a.config, a.n)
    levels = []
    state = {"last": None}
    bounds = [32, 64, 128, 256, 512, 1024, 2048, 4096, 1 << 40]

    def audit(side, lo, hi, depth):
        key = id(side)
        if state["last"] != key:
            state["last"] = key
            levels.append(collections.Counter())
        sz = hi - lo
        cls = next(b for b in bounds if sz <= b)
        levels[-1][(cls, "segs")] += 1
        levels[-1][(cls, "strs")] += sz
        levels[-1][("depth", "max")] = max(levels[-1][("depth", "max")], depth)

    audited_sort(arena, h.copy(), 0, SampleSortConfig(), None, audit, None)
    for i, c in enumerate(levels):
        row = " ".join(f"<={b if b < 1 << 40 else 'inf'}:{c[(b, 'segs')]}/{c[(b, 'strs')]}"
                       for b in bounds if c[(b, "segs")])
        print(f"level {i + 1}: maxdepth {c[('depth', 'max')]}  {row}")


if __name__ == "__main__":
    main()
