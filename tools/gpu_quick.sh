cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_gemm.py 32768 272 5 nn 2>&1 | tail -2
timeout 300 python tools/profile_gemm.py 32768 272 5 tn 2>&1 | tail -2
PSD_GEMM=legacy timeout 300 python tools/profile_gemm.py 32768 272 3 nn 2>&1 | tail -2
timeout 300 python tools/probe_c3.py 2>&1 | tail -12
