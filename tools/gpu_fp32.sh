cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_fp32.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_fp32.log
timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 > gpurun_out/probe_fp32.log 2>&1; echo "probe rc=$?"
tail -10 gpurun_out/probe_fp32.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fp32.csv python tools/probe_c3.py 32768 256 16 1 fp32 > gpurun_out/ncu_fp32.log 2>&1; echo "ncu rc=$?"
