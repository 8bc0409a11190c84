cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -2 /tmp/pt.log
for st in 1 0; do
PSD_STAGED_EPI=$st timeout 300 python tools/probe_c3.py 32768 256 16 1 > /tmp/o.log 2>&1; grep -E "recon|total" /tmp/o.log | sed "s/^/staged=$st /"
done
