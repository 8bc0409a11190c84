cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_chol.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_chol.log
timeout 300 python tools/probe_c3.py 32768 256 16 1 > gpurun_out/probe64_t.log 2>&1; echo "probe rc=$?"
grep -E "qr |total|eigh|recon|sketch" gpurun_out/probe64_t.log
timeout 300 python tools/probe_c3.py 8192 128 16 2 > gpurun_out/probe_c2.log 2>&1; echo "probe rc=$?"
grep -E "proj 2|qr |total|eigh|recon|sketch" gpurun_out/probe_c2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fp64.csv python tools/probe_c3.py 32768 256 16 1 > gpurun_out/ncu_fp64.log 2>&1; echo "ncu rc=$?"
