#!/bin/bash
# oversampling factor of the wide steps' samples, interleaved with the default
mkdir -p gpurun_out
for r in 1 2; do for c in 2 3 4 5; do for o in "" "--cfg alpha=2"; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline $o 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());print($c,'$o',round(d['ms_per_step'],4),d['levels'])" >> gpurun_out/sweep_alpha.txt
done; done; done
