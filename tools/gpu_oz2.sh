cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/probe_c3.py 32768 256 16 1 2>&1 | grep -E "proj 2|sketch|int8|total"; done
