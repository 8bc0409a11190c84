cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log; grep -E "^FAILED" gpurun_out/pt.log | head
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.log'))
print('value', d['value'], d['step_ms_min_median_max']); print('e2e', d['e2e']['value']); print('roof', d['roofline']['bound'], d['roofline']['frac'], d['roofline']['achieved'], d['roofline']['peak']); print(d['stages_ms_per_projection']); print('clocks', d['clocks']); print('fp32', d['fp32']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
