cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -4
