"""Key per-kernel metrics from an `ncu --set full` report (run here, no GPU needed).

    python profiles/ncu_summary.py gpurun_out/prof_cfg2.ncu-rep [--json out.json]

Reads `ncu -i <rep> --page raw --csv` and prints, per profiled launch: device
time, DRAM bytes read/written (the `traffic` of bench.py's roofline object),
DRAM throughput, L2 hit rate, achieved occupancy, SM throughput and registers.
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "lts__t_bytes.sum": "l2_bytes",
    "smsp__inst_executed.sum": "inst",
}

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9,
        "us": 1e-6, "ms": 1e-3}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(header, r))
        u = dict(zip(header, units))
        rec = {"kernel": re.sub(r"\(.*", "", d.get("Kernel Name", "?"))[:60],
               "id": d.get("ID")}
        for m, short in METRICS.items():
            if m in d and d[m] not in ("", "n/a"):
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    continue
                rec[short] = v * UNIT.get(u.get(m, ""), 1)
        res.append(rec)
    return res


def main():
    rep = sys.argv[1]
    recs = load(rep)
    for r in recs:
        t = r.get("time", 0)
        rd, wr = r.get("dram_read", 0), r.get("dram_write", 0)
        gbs = (rd + wr) / t / 1e9 if t else 0
        print(f"{r['kernel']:40s} {t * 1e3:8.3f} ms  dram R {rd / 1e6:8.1f} MB  W {wr / 1e6:8.1f} MB"
              f"  {gbs:7.0f} GB/s ({r.get('dram_pct', 0):4.1f}%)  L2hit {r.get('l2_hit_pct', 0):5.1f}%"
              f"  occ {r.get('occupancy_pct', 0):5.1f}%  sm {r.get('sm_pct', 0):5.1f}%"
              f"  regs {r.get('regs', 0):.0f}")
    if "--json" in sys.argv:
        json.dump(recs, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
