cd $GRAFT_REPO_ROOT
PSD_CHOL_TIMERS=1 timeout 300 python tools/probe_c3.py 8192 256 16 1 2>&1 | grep -E "chol|proj 2|qr "  | head -12
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
