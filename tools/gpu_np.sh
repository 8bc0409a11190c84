cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_ozaki.py 2>&1 | tail -6
PSD_FP64_OZAKI=1 timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > /tmp/pt.log 2>&1; echo "pytest(ozaki) rc=$?"; tail -1 /tmp/pt.log; grep -E "^FAILED" /tmp/pt.log | head -8
PSD_FP64_OZAKI=1 timeout 300 python tools/probe_c3.py 32768 256 16 1 > /tmp/o.log 2>&1; grep -E "proj 2|sketch|total" /tmp/o.log
PSD_FP64_OZAKI=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_oz.csv python tools/probe_c3.py 32768 256 16 1 > /dev/null 2>&1; echo ncu=$?
