# Jacobi: deferred V accumulation (rotation log) vs per-step V update
for D in 0 1; do echo "deferv=$D"; PSD_JACOBI_DEFERV=$D PSD_JACOBI_TRACE=gpurun_out/jt_d$D.bin timeout 100 python tools/probe_eigh.py 272 2 2>&1 | tail -1; python tools/jacobi_trace.py gpurun_out/jt_d$D.bin | tail -2; PSD_JACOBI_DEFERV=$D timeout 100 python tools/probe_eigh.py 272 4 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "eigh or golden or config3_shape or exact" 2>&1 | tail -1
