#!/bin/bash
# A/B timing of two builds of libs5.so on one box (interleaved, 3 rounds):
#   build the variant to paper_1305_1157_b200/libs5_base.so, then
#   /usr/local/graft/bin/gpurun --timeout 1200 -- 'bash profiles/ab.sh 3 4 5'
# _lib.py loads $S5_LIB instead of the in-tree libs5.so when it is set.
mkdir -p gpurun_out
CFGS=${@:-2 3 4 5}
for r in 1 2 3; do for c in $CFGS; do for L in base new; do
  if [ $L = base ]; then export S5_LIB=$PWD/paper_1305_1157_b200/libs5_base.so; else unset S5_LIB; fi
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$L',$c,d['ms_per_step'])" >> gpurun_out/ab.txt
done; done; done
