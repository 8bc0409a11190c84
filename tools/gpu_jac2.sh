cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 120 python tools/probe_eigh.py 272 4 2>&1 | tail -1; done
timeout 120 python tools/probe_eigh.py 144 3 2>&1 | tail -1
timeout 120 python tools/probe_eigh.py 1000 2 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/probe_c3.py 32768 256 16 1 2>&1 | grep -E "proj 2|eigh|total"
