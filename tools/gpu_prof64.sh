cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_CHOL_TIMERS=1 PSD_JACOBI_TIMERS=1 timeout 300 python tools/probe_c3.py 32768 256 16 1 > gpurun_out/probe64_t.log 2>&1; echo "probe rc=$?"
grep -E "chol m|jacobi" gpurun_out/probe64_t.log | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fp64.csv python tools/probe_c3.py 32768 256 16 1 > gpurun_out/ncu_fp64.log 2>&1; echo "ncu rc=$?"
