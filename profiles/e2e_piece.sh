#!/bin/bash
# e2e (host numpy buffers) of config 2 for several staging piece sizes
# (S5_HOST_PIECE elements per pinned staging piece), interleaved, one box
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
rm -f gpurun_out/e2e_piece.txt
for r in 1 2; do for P in ${PIECES:-1048576 2097152 4194304 8388608}; do
  S5_HOST_PIECE=$P python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());e=d['e2e'];print($P,round(e['ms_per_step'],3),{k:round(v,3) for k,v in e['phases_ms'].items() if 'bytes' not in k})" >> gpurun_out/e2e_piece.txt
done; done
cat gpurun_out/e2e_piece.txt
