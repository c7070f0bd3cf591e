#!/bin/bash
# ncu --set full of one sort per config (kernels of the wide and local tiers),
# summarised on the box (the .ncu-rep files are too large to bring back):
# per-launch table + JSON (ncu_summary.py) and warp-stall samples by source
# line of the main kernels (stall_by_line.py).  Usage (gpurun box):
#   bash profiles/capture_cfgs.sh "2 3 4 5" [tag]
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CFGS=${1:-"2 3 4 5"}; TAG=${2:-r02}
REP=/tmp/ncu_$TAG; mkdir -p $REP
for C in $CFGS; do
  python profiles/profile_one.py --config $C > /dev/null || exit 1
  timeout 900 ncu --set full --import-source on --clock-control none -f \
      -k regex:"k_local|k_wide_scatter|k_wide_count|k_small|k_narrow" --launch-count 48 \
      -o $REP/full_cfg$C python profiles/profile_one.py --config $C \
      > gpurun_out/${TAG}_ncu_cfg$C.log 2>&1
  echo "cfg $C rc=$?"
  python profiles/ncu_summary.py $REP/full_cfg$C.ncu-rep --json gpurun_out/${TAG}_ncu_cfg$C.json \
      > gpurun_out/${TAG}_ncu_cfg$C.txt 2>&1
  for K in "k_local_w" "k_local.*int.64," "k_local.*int.128," "k_local.*int.256," "k_local.*int.512," \
           "k_wide_scatter" "k_wide_count" "k_narrow"; do
    echo "== $K" >> gpurun_out/${TAG}_stalls_cfg$C.txt
    timeout 300 python profiles/stall_by_line.py $REP/full_cfg$C.ncu-rep "$K" 0 \
        >> gpurun_out/${TAG}_stalls_cfg$C.txt 2>&1
  done
done
ls -la gpurun_out/
