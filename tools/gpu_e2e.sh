cd $GRAFT_REPO_ROOT
timeout 120 python -X faulthandler -c "
import torch; torch.zeros(1, device='cuda')
import bench, time
s = bench.ClockSampler(0); s.start(); time.sleep(1); print(s.stop())
" 2>&1 | tail -15
timeout 900 python -X faulthandler bench.py --no-fp32 --no-cpu-baseline --steps 6 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -30 gpurun_out/bench.err
