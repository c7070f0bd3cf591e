set -x
nvidia-smi -L
export PYTHONDONTWRITEBYTECODE=1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python profiles/sanitize.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python profiles/sanitize.py --quick > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python profiles/sanitize.py --quick > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.log
for c in 3 4 5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2base_cfg$c.json 2> gpurun_out/r2base_cfg$c.err; done
tail -3 gpurun_out/san_*.log
