cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 600 python tools/probe_c3.py > gpurun_out/probe.log 2>&1
echo "probe rc=$?"
tail -60 gpurun_out/pytest_gpu.log
cat gpurun_out/probe.log
