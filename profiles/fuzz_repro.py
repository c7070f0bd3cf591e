"""One seed of tests/test_gpu_fuzz.py with configuration overrides (key=value ...): first mismatches against the oracle."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import oracle as O
from paper_1305_1157_b200 import arena_from_strings, sort_with_lcp
import test_gpu_fuzz as F
seed = int(sys.argv[1])
rng = np.random.default_rng(1000 + seed)
strs = F._strings(rng); cfg = F._config(rng)
for k, v in [a.split("=") for a in sys.argv[2:]]:
    setattr(cfg, k, int(v) if v.lstrip('-').isdigit() else v)
arena, h0 = arena_from_strings(strs)
want = h0.copy(); O.parallel_sample_sort(arena, want, 4)
got = h0.copy(); _, lcp = sort_with_lcp(arena, got, cfg=cfg)
wl = O.adjacent_lcps(arena, want)
bad = np.nonzero(lcp != wl)[0]
print("lib", os.environ.get("S5_LIB", "new"), "n", len(strs), "perm", np.array_equal(np.sort(got), np.sort(h0)), "order", O.contents_equal(arena, got, want), "bad lcps", bad.size, bad[:10])
for i in bad[:2]:
    print(i, "got", lcp[i], "want", wl[i], arena.string_at(int(got[i]))[:60], arena.string_at(int(got[i+1]))[:60])
