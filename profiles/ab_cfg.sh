#!/bin/bash
# A/B of a configuration override on one build (interleaved, R rounds):
#   bash profiles/ab_cfg.sh "narrow_max=262144 wide_v=255" 2 3 4 5
# prints "A|B config ms" lines into gpurun_out/ab_cfg.txt
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
OV=$1; shift; CFGS=${@:-2 3 4 5}; R=${R:-2}
ARGS=""; for kv in $OV; do ARGS="$ARGS --cfg $kv"; done
for r in $(seq $R); do for c in $CFGS; do for L in A B; do
  if [ $L = A ]; then X=""; else X="$ARGS"; fi
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline $X 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$L',$c,round(d['ms_per_step'],4),d['levels'],{k:round(v,3) for k,v in d['kernels_ms_per_step'].items() if v>0.02})" >> gpurun_out/ab_cfg.txt
done; done; done
cat gpurun_out/ab_cfg.txt
