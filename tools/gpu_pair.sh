cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/probe_tc32.py 4096 > gpurun_out/tc32_pair.log 2>&1; echo "probe rc=$?"; grep -E "ALL OK|FAIL|Error|error" gpurun_out/tc32_pair.log | head -3
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 > gpurun_out/probe_fp32.log 2>&1; echo "probe32 rc=$?"
grep -E "symcheck|sketch|qr |eigh|recon|total" gpurun_out/probe_fp32.log
