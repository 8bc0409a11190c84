cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for kc in 0 4096 2048 1024; do PSD_TC32_KCHUNK=$kc timeout 300 python tools/probe_fp32_fullsize.py 32768 2>&1 | tail -1; done
for kc in 0 2048 1024; do PSD_TC32_KCHUNK=$kc timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 2>&1 | grep -E "sketch_gemm|total"; done
