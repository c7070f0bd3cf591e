# gpurun payload: GPU tests + default bench (writes gpurun_out/)
#   bash profiles/run_check.sh [pytest -m expression] [bench args...]
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
M="${1:-gpu and not slow}"; shift || true
timeout 1500 python -m pytest tests -q -x -m "$M" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
if [ "$#" -gt 0 ]; then
  timeout 900 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 400 gpurun_out/bench.err
  python profiles/show_bench.py gpurun_out/bench.json
fi
