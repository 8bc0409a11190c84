cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > /tmp/pt.log 2>&1; echo "run $i rc=$?"; tail -1 /tmp/pt.log; grep -E "^FAILED" /tmp/pt.log | head -3
done
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "reduced_n" 2>&1 | tail -1; done
