cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fp32.py -q --timeout 600 -p no:cacheprovider -x > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -2 /tmp/pt.log
timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 > /tmp/o.log 2>&1; grep -E "symcheck|total" /tmp/o.log
