cd $GRAFT_REPO_ROOT
PSD_JACOBI_TIMERS=1 timeout 300 python tools/probe_eigh.py 64 2 2>&1
PSD_JACOBI_TIMERS=1 timeout 300 python tools/probe_eigh.py 272 3 2>&1
PSD_JACOBI_TIMERS=1 timeout 300 python tools/probe_eigh.py 544 2 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
