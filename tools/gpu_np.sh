cd $GRAFT_REPO_ROOT
timeout 120 python tools/probe_tc32.py 4096 2>&1 | grep -E "rel err|ALL|FAIL|rror" | head -12
timeout 900 python -m pytest tests/test_gpu_fp32.py -q --timeout 600 -p no:cacheprovider -x > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -3 /tmp/pt.log
for ts in 1 0; do
PSD_TC32_TS=$ts timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 > /tmp/o.log 2>&1; grep -E "sketch_gemm |total" /tmp/o.log | sed "s/^/ts=$ts /"
done
