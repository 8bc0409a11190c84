cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 120 python tools/probe_eigh.py 272 4 2>&1 | tail -1; done
timeout 120 python tools/probe_eigh.py 144 3 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
