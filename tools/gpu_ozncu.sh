cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"residues_rows_mma" --launch-skip 5 -c 1 -o gpurun_out/oz_resmma python tools/probe_ozaki.py > gpurun_out/oz_ncu.log 2>&1; echo ncu=$?
