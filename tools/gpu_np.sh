cd $GRAFT_REPO_ROOT
timeout 120 python tools/probe_tc32.py 4096 2>&1 | grep -E "ALL OK|FAIL"
for pf in 0 4 8 16; do
PSD_TC32_PF=$pf timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 2>&1 | grep -E "sketch_gemm " | sed "s/^/pf=$pf /"
done
PSD_TC32_PF=8 PSD_TC32_NPROD=1 timeout 300 python tools/probe_c3.py 32768 256 16 1 fp32 2>&1 | grep -E "sketch_gemm " | sed "s/^/pf=8 nprod1 /"
