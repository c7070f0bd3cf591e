#!/bin/bash
# Interleaved timing of several builds of libs5.so on one box:
#   LIBS="base b new" CFGS="2 4 5" R=3 bash profiles/abn.sh
# "new" = the in-tree libs5.so; any other name X = paper_1305_1157_b200/libs5_X.so
# (_lib.py loads $S5_LIB instead of the in-tree library when it is set).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
LIBS=${LIBS:-"base new"}; CFGS=${CFGS:-"2 3 4 5"}; R=${R:-3}
for r in $(seq $R); do for c in $CFGS; do for L in $LIBS; do
  if [ $L = new ]; then unset S5_LIB; else export S5_LIB=$PWD/paper_1305_1157_b200/libs5_$L.so; fi
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$L',$c,round(d['ms_per_step'],4))" >> gpurun_out/abn.txt
done; done; done
python - <<'PY'
import collections
d = collections.defaultdict(list)
for ln in open("gpurun_out/abn.txt"):
    L, c, ms = ln.split()
    d[(int(c), L)].append(float(ms))
for (c, L), v in sorted(d.items()):
    print(f"cfg {c} {L:6s} median {sorted(v)[len(v)//2]:.4f}  all {v}")
PY
