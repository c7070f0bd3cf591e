"""e2e (public API, numpy host buffers) of one config under several host
staging settings, interleaved in one process per setting.

    python profiles/e2e_ring.py [config] [steps]   (on a gpurun box)

Each setting is a child process with its own S5_HOST_RING / S5_RING_PIECE /
S5_RING_SLOTS (read once per device by libs5.so); lines of
"setting  e2e_ms  h2d  sort  d2h" are printed, two interleaved rounds.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SETTINGS = [
    {"S5_HOST_RING": "0"},
    {"S5_HOST_RING": "1", "S5_RING_PIECE": str(1 << 20), "S5_RING_SLOTS": "32"},
    {"S5_HOST_RING": "1", "S5_RING_PIECE": str(1 << 20), "S5_RING_SLOTS": "64"},
    {"S5_HOST_RING": "1", "S5_RING_PIECE": str(2 << 20), "S5_RING_SLOTS": "32"},
    {"S5_HOST_RING": "3", "S5_RING_PIECE": str(2 << 20), "S5_RING_SLOTS": "48"},
    {"S5_HOST_RING": "7", "S5_RING_PIECE": str(1 << 20), "S5_RING_SLOTS": "64"},
]

CHILD = r"""
import json, sys, time
sys.path.insert(0, %r)
import numpy as np, torch
import bench
from paper_1305_1157_b200 import samplesort as ss
arena, h0, _ = bench.workload(%d, None)
cfg = ss.SampleSortConfig()
ms, ph = bench.measure_e2e(arena, h0, cfg, %d, 3)
print(json.dumps({"ms": ms * 1e3, "phases": ph}))
"""


def main():
    config = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    for rnd in range(2):
        for s in SETTINGS:
            env = dict(os.environ, **s)
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, config, steps)], env=env,
                                 capture_output=True, text=True)
            tag = " ".join(f"{k[3:]}={v}" for k, v in s.items())
            if out.returncode:
                print(tag, "FAILED", out.stderr[-500:], flush=True)
                continue
            d = json.loads(out.stdout.strip().splitlines()[-1])
            p = d["phases"]
            print(f"r{rnd} {tag:45s} e2e {d['ms']:7.3f}  h2d {p['h2d']:6.3f}  sort {p['sort']:6.3f}  "
                  f"d2h {p['d2h']:6.3f}", flush=True)


if __name__ == "__main__":
    main()
