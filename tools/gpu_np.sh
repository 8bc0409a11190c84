cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_ozaki.py 2>&1 | tail -6
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -1 /tmp/pt.log; grep -E "^FAILED" /tmp/pt.log | head -8
timeout 300 python tools/probe_c3.py 32768 256 16 1 > /tmp/o.log 2>&1; grep -E "proj 2|ms/proj" /tmp/o.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_oz.csv python tools/probe_c3.py 32768 256 16 1 > /dev/null 2>&1; echo ncu=$?
