"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python profiles/summarize_launches.py gpurun_out/launches_cfg2.csv [--only s5::]

Prints launches, total and mean device time per kernel and its share of the
total.  ncu times are cold-cache and serialised: compare SHARES with the
CUDA-event numbers of bench.py, not absolute values.
"""
import csv
import re
import sys
from collections import defaultdict


def load(path):
    rows = []
    with open(path, newline="") as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "nsecond": 1e-6, "second": 1e3}.get(unit, 1e-6)
        rows.append((r["Kernel Name"], val * scale))
    return rows


def short(name):
    m = re.search(r"(k_[a-z0-9_]+)", name)
    return m.group(1) if m else name[:60]


def main():
    path = sys.argv[1]
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    rows = load(path)
    agg = defaultdict(lambda: [0, 0.0])
    for name, ms in rows:
        if only and only not in name:
            continue
        k = short(name)
        agg[k][0] += 1
        agg[k][1] += ms
    total = sum(v[1] for v in agg.values())
    print(f"{'kernel':32s} {'launches':>9s} {'total ms':>10s} {'mean ms':>9s} {'share':>7s}")
    for k, (cnt, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:32s} {cnt:9d} {ms:10.3f} {ms / cnt:9.4f} {100 * ms / total:6.1f}%")
    print(f"{'TOTAL':32s} {sum(v[0] for v in agg.values()):9d} {total:10.3f}")


if __name__ == "__main__":
    main()
