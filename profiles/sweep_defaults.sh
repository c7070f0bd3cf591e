#!/bin/bash
mkdir -p gpurun_out
for c in 2 3 4; do
for o in "" "--cfg wide_target=1024" "--cfg wide_target=256" "--cfg wide_v=1023" "--cfg wide_v=255" "--cfg alpha=8" "--cfg local_max=2048 --cfg wide_target=256"; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline $o 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());print($c,'$o',round(d['ms_per_step'],4),d['levels'])" >> gpurun_out/sweep.txt
done; done
