cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_c3.py 1000 40 10 2 > /tmp/o.log 2>&1; grep -E "eigh|total" /tmp/o.log
PSD_JACOBI_SMALL=0 timeout 300 python tools/probe_c3.py 1000 40 10 2 > /tmp/o.log 2>&1; grep -E "eigh|total" /tmp/o.log | sed 's/^/block: /'
