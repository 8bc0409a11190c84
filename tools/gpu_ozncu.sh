cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_ozaki.py 2>&1 | tail -1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"residues_rows" --launch-skip 5 -c 1 -o gpurun_out/oz_res3 python tools/probe_ozaki.py > gpurun_out/oz_ncu.log 2>&1; echo ncu=$?
