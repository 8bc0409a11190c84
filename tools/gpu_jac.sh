cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q --timeout 200 -p no:cacheprovider -x -k "eigh or jacobi" > gpurun_out/pytest_jac.log 2>&1
echo "pytest-eigh rc=$?"; tail -3 gpurun_out/pytest_jac.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
PSD_JACOBI_TIMERS=1 timeout 300 python tools/probe_c3.py 32768 256 16 1 > gpurun_out/probe64_t.log 2>&1; echo "probe rc=$?"
grep -E "jacobi|eigh|total" gpurun_out/probe64_t.log | tail -4
timeout 300 python tools/probe_c3.py 8192 128 16 2 > gpurun_out/probe_c2.log 2>&1; echo "probe rc=$?"
grep -E "proj 2|eigh|total" gpurun_out/probe_c2.log
