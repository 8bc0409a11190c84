cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -3 /tmp/pt.log
timeout 300 python tools/probe_c5b.py 2>&1 | tail -1
timeout 300 python tools/probe_c3.py 1000 40 10 2 > /tmp/o.log 2>&1; grep -E "eigh|total" /tmp/o.log
