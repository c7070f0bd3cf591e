#!/bin/bash
# One round's profile capture on a gpurun box (1 GPU).  Usage:
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash profiles/capture.sh 2'
# Outputs under gpurun_out/ (summarised here with summarize_launches.py,
# ncu_summary.py, stall_by_line.py into profiles/rNN_*):
#   bench_cfgC.json     bench line without ncu (the number that counts)
#   launches_cfgC.csv   ncu launch list of the same bench command
#   full_cfgC.ncu-rep   ncu --set full of one sort (profile_one.py)
#   libs5_prof.so       the library that was profiled (line info for the source page)
set -e
C=${1:-2}
mkdir -p gpurun_out
python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$C.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg$C.csv \
    python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python profiles/profile_one.py --config $C > /dev/null
ncu --set full --import-source on --clock-control none -f -o gpurun_out/full_cfg$C \
    python profiles/profile_one.py --config $C > gpurun_out/ncu_full.log 2>&1
cp paper_1305_1157_b200/libs5.so gpurun_out/libs5_prof.so
echo captured
