cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 120 python tools/probe_eigh.py 272 4 2>&1 | tail -1; done
PSD_JACOBI_TIMERS=1 timeout 120 python tools/probe_eigh.py 272 2 2>&1 | tail -2
