#!/bin/bash
# A round's evidence on one gpurun box:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash profiles/capture_round.sh r02'
# 1. the default bench line (config 2 headline + configs 3-5 + CPU baseline)
# 2. the ncu launch list of the config-2 bench command (gpu__time_duration)
# 3. ncu --set full of one sort per config, summarised on the box
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TAG=${1:-r02}
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_cfg2.csv \
    python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config \
    > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
bash profiles/capture_cfgs.sh "2 3 4 5" $TAG
