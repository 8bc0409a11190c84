cd $GRAFT_REPO_ROOT
PSD_CHOL_TIMERS=1 timeout 300 python tools/probe_c3.py 8192 256 16 1 2>&1 | grep "chol m=" | tail -3
