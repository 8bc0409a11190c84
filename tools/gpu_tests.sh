cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 > gpurun_out/probe_fp32.log 2>&1; echo "probe rc=$?"
tail -10 gpurun_out/probe_fp32.log
