cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 > gpurun_out/probe_fp32.log 2>&1 || { echo "probe failed"; exit 1; }
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"tc32_gemm2_kernel" -s 4 -c 1 -o gpurun_out/tc32_pair2 python tools/probe_c3.py 32768 256 16 1 fp32 > gpurun_out/ncu_tc32.log 2>&1; echo "ncu rc=$?"
