"""Wide segments by the common-prefix length of their keys, per level (audit hook).

    python profiles/prefix_stats.py 3

How many strings sit in multi-CTA segments whose keys at the segment depth
all share L leading bytes (L = 8: all keys equal) -- the levels a
common-prefix skip in the wide tier would save."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1305_1157_b200 import datasets
from paper_1305_1157_b200._audit import audited_sort
from paper_1305_1157_b200.samplesort import SampleSortConfig
cfgn = int(sys.argv[1])
arena, h = datasets.generate(cfgn)
data = arena.data
levels = []
state = {"last": None}
def keys_at(offs, depth):
    out = np.zeros(offs.size, np.uint64)
    term = np.zeros(offs.size, bool)
    for b in range(8):
        byte = data[offs + depth + b].astype(np.uint64)
        byte[term] = 0
        term |= byte == 0
        out |= byte << np.uint64(56 - 8 * b)
    return out
def audit(side, lo, hi, depth):
    key = id(side)
    if state["last"] != key:
        state["last"] = key
        levels.append(collections.Counter())
    sz = hi - lo
    if sz <= 4096: return
    offs = side[lo:hi]
    k = keys_at(offs, depth)
    mn, mx = int(k.min()), int(k.max())
    x = mn ^ mx
    L = 8 if x == 0 else (64 - x.bit_length()) // 8
    levels[-1][L] += sz
audited_sort(arena, h.copy(), 0, SampleSortConfig(), None, audit, None)
for i, c in enumerate(levels):
    print(f"level {i+1}: wide strings by common-prefix bytes: " + " ".join(f"L{L}:{c[L]}" for L in sorted(c)))
