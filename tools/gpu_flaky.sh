cd $GRAFT_REPO_ROOT
timeout 900 python tools/flaky.py 4096 60 2>&1 | grep -E "BAD" | tail -2
for i in 1 2 3; do
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > /tmp/pt.log 2>&1; echo "run $i rc=$?"; tail -1 /tmp/pt.log; grep -E "^FAILED" /tmp/pt.log | head -3
done
timeout 300 python tools/probe_c3.py 32768 256 16 1 > /tmp/o.log 2>&1; grep -E "recon|total" /tmp/o.log
timeout 300 python tools/probe_c3.py 8192 128 16 2 > /tmp/o.log 2>&1; grep -E "sketch|total" /tmp/o.log
