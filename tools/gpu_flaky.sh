cd $GRAFT_REPO_ROOT
for i in 1 2 3 4; do
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > /tmp/pt.log 2>&1; echo "run $i rc=$?"; tail -1 /tmp/pt.log; grep -E "^FAILED" /tmp/pt.log | head -3
done
