#!/bin/bash
# A/B/n timing of several builds of libs5.so on one box (interleaved, 3 rounds):
#   /usr/local/graft/bin/gpurun -- 'bash profiles/abn.sh "2 5" base new v3'
# "new" is the in-tree libs5.so; any other name X loads paper_1305_1157_b200/libs5_X.so.
mkdir -p gpurun_out
CFGS=$1; shift
for r in 1 2 3; do for c in $CFGS; do for L in "$@"; do
  if [ $L = new ]; then unset S5_LIB; else export S5_LIB=$PWD/paper_1305_1157_b200/libs5_$L.so; fi
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());k=d.get('kernels_ms_per_step',{});print('$L',$c,round(d['ms_per_step'],4),k.get('k_wide_count'))" >> gpurun_out/abn.txt
done; done; done
