cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -q -x -m "gpu and not slow" > gpurun_out/c3_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c3_tests.log; tail -3 gpurun_out/c3_tests.log
timeout 300 ncu --metrics dram__bytes_write.sum,dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_op_write.sum profiles/probes/write_probe > gpurun_out/c3_probe.txt 2>&1; echo probe rc=$?
rm -f gpurun_out/ab.txt; timeout 1500 bash profiles/ab.sh 2 3 4 5; cat gpurun_out/ab.txt
