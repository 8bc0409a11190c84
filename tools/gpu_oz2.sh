cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_ozaki.py 2>&1 | tail -6
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_oz.csv python tools/probe_c3.py 32768 256 16 1 > /dev/null 2>&1; echo ncu=$?
