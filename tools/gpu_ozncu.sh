cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_ozaki.py 2>&1 | tail -2 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"residues_rows|i8_gemm2|crt_kernel" --launch-skip 15 -c 3 -o gpurun_out/oz_full2 python tools/probe_ozaki.py > gpurun_out/oz_ncu.log 2>&1; echo ncu=$?
