cd $GRAFT_REPO_ROOT
for ns in 0 1 2 0 1; do echo "nsplit=$ns"; PSD_OZ_NSPLIT=$ns timeout 300 python tools/probe_c3.py 32768 256 16 1 2>&1 | grep -E "int8_gemm|total"; done
