cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSD_JACOBI_TIMERS=1 timeout 300 python tools/probe_c3.py 32768 256 16 1 > gpurun_out/probe64_t.log 2>&1; echo "probe rc=$?"
grep -E "jacobi|eigh" gpurun_out/probe64_t.log | tail -2
timeout 300 python -m pytest tests -m gpu -q --timeout 200 -p no:cacheprovider -x -k "eigh or golden or config" 2>&1 | tail -2
