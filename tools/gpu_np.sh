cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -3 /tmp/pt.log
timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 > /tmp/o.log 2>&1; grep -E "sketch|total|symcheck|qr |eigh|recon" /tmp/o.log
timeout 300 python tools/probe_fp32_fullsize.py 32768 2>&1 | tail -1
