#!/bin/bash
# A/B of an environment override (e.g. S5_WIDE_CHUNK=8192) on one build:
#   bash profiles/ab_env.sh "S5_WIDE_CHUNK=8192" 2 5
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
KV=$1; shift; CFGS=${@:-2 5}; R=${R:-2}
for r in $(seq $R); do for c in $CFGS; do for L in A B; do
  if [ $L = A ]; then E=""; else E="$KV"; fi
  env $E python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-per-config 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$L','$E',$c,round(d['ms_per_step'],4),{k:round(v,3) for k,v in d['kernels_ms_per_step'].items() if k in ('k_wide_count','k_wide_scatter')})" >> gpurun_out/ab_env.txt
done; done; done
