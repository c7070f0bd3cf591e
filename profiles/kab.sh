mkdir -p gpurun_out; rm -f gpurun_out/kab.txt
for c in ${CFGS:-2 5}; do for L in base new base new; do
  if [ $L = base ]; then export S5_LIB=$PWD/paper_1305_1157_b200/libs5_base.so; else unset S5_LIB; fi
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-per-config 2>/dev/null |
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$L',$c,round(d['ms_per_step'],4),{k:round(v,3) for k,v in d['kernels_ms_per_step'].items() if v>0.02})" >> gpurun_out/kab.txt
done; done
cat gpurun_out/kab.txt
