#!/bin/bash
# ncu --set full of one sort, summarised on the box: per-launch table and
# stall-by-line of the named kernels.  Usage (gpurun box):
#   bash profiles/capture_kern.sh TAG CONFIG "kernel-regex ..." [--cfg key=value ...]
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=$1; C=$2; KS=$3; shift 3
REP=/tmp/ncu_$TAG; mkdir -p $REP
python profiles/profile_one.py --config $C "$@" > /dev/null || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -f \
    -k regex:"k_local|k_wide|k_small|k_narrow" --launch-count 64 \
    -o $REP/full python profiles/profile_one.py --config $C "$@" > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
python profiles/ncu_summary.py $REP/full.ncu-rep --json gpurun_out/${TAG}_ncu.json > gpurun_out/${TAG}_ncu.txt 2>&1
for K in $KS; do
  echo "== $K" >> gpurun_out/${TAG}_stalls.txt
  timeout 300 python profiles/stall_by_line.py $REP/full.ncu-rep "$K" 0 >> gpurun_out/${TAG}_stalls.txt 2>&1
done
