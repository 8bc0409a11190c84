cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_JACOBI_TIMERS=1 timeout 300 python tools/probe_c3.py 32768 256 16 1 > gpurun_out/probe64_t.log 2>&1; echo "probe rc=$?"
grep -E "jacobi|eigh" gpurun_out/probe64_t.log | tail -3
