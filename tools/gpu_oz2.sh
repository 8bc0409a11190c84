cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ozaki.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_oz.csv python tools/probe_c3.py 32768 256 16 1 > /dev/null 2>&1; echo ncu=$?
