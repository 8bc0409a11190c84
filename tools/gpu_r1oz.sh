cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pt_int8.log 2>&1; echo "pytest(int8 default) rc=$?"; tail -1 gpurun_out/pt_int8.log; grep -E "^FAILED|Error" gpurun_out/pt_int8.log | head -8
PSD_FP64_OZAKI=0 timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pt_dmma.log 2>&1; echo "pytest(dmma) rc=$?"; tail -1 gpurun_out/pt_dmma.log; grep -E "^FAILED" gpurun_out/pt_dmma.log | head -8
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
