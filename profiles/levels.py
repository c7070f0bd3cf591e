"""Per-level kernel times from bench.py --launch-recs JSON lines.

    python profiles/levels.py gpurun_out/bench_cfg4.json [...]
"""
import collections
import json
import sys

for path in [a for a in sys.argv[1:] if not a.startswith('--')]:
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    print(f"{path}: {d['ms_per_step']:.3f} ms/step")
    agg = collections.defaultdict(lambda: [0.0, 0])
    recs = d.get("launch_recs") or []
    for r in recs:
        k, lvl, n, ms = r[:4]
        agg[(lvl, k)][0] += ms
        agg[(lvl, k)][1] += n
    for (lvl, k), (ms, n) in sorted(agg.items()):
        if ms > 0.02:
            ps = f"{1e9 * ms / n:7.1f} ps/string" if n else ""
            print(f"   L{lvl} {k:16s} {ms:7.3f} ms {n / 1e6:8.2f} M {ps}")
    if recs and len(recs[0]) > 4 and "--timeline" in sys.argv:
        # serial (profiling-mode) timeline: idle gaps between consecutive launches
        busy = sum(r[3] for r in recs)
        end = max(r[4] + r[3] for r in recs)
        print(f"   timeline: {end:.3f} ms, kernels busy {busy:.3f} ms, gaps {end - busy:.3f} ms")
        for a, b in zip(recs, recs[1:]):
            gap = b[4] - (a[4] + a[3])
            if gap > 0.01:
                print(f"     gap {gap:.3f} ms before L{b[1]} {b[0]}")
