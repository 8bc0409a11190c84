cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider 2>&1 | tail -2
timeout 1500 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/c4.log 2> gpurun_out/c4.err; echo "c4 rc=$?"; tail -3 gpurun_out/c4.err; cat gpurun_out/c4.log
