"""Print the key numbers of bench.py JSON lines: python profiles/show_bench.py f1.json ..."""
import json
import sys

for path in sys.argv[1:]:
    lines = [ln for ln in open(path).read().strip().splitlines() if ln.startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    w = d["config"]["workload"].split(":")[0]
    print(f"{path}: {w} {d['ms_per_step']:.3f} ms/step  {d['value'] / 1e9:.3f} Gstr/s  "
          f"e2e {d['e2e']['ms_per_step']:.1f} ms  levels {d['levels']}  "
          f"sort-roofline {d['roofline_sort']['frac']:.3f}  dom {d['roofline']['kernel']} "
          f"{d['roofline']['frac']:.3f}")
    print("   kernels:", {k: v for k, v in d["kernels_ms_per_step"].items() if v > 0.01})
    print("   n_p:", d["n_per_pass"])
