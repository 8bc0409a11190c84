cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/probe_tc32.py 16384 > gpurun_out/tc32.log 2>&1; echo "rc=$?" >> gpurun_out/tc32.log
cat gpurun_out/tc32.log | tail -20
