"""Per-level kernel times from bench.py --launch-recs JSON lines.

    python profiles/levels.py gpurun_out/bench_cfg4.json [...]
"""
import collections
import json
import sys

for path in sys.argv[1:]:
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    print(f"{path}: {d['ms_per_step']:.3f} ms/step")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for k, lvl, n, ms in d.get("launch_recs") or []:
        agg[(lvl, k)][0] += ms
        agg[(lvl, k)][1] += n
    for (lvl, k), (ms, n) in sorted(agg.items()):
        if ms > 0.02:
            ps = f"{1e9 * ms / n:7.1f} ps/string" if n else ""
            print(f"   L{lvl} {k:16s} {ms:7.3f} ms {n / 1e6:8.2f} M {ps}")
