cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log; grep -E "^FAILED|Error" gpurun_out/pt.log | head -8
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.log'))
print('value', d['value'], 'ms', d['ms_per_step'], d['step_ms_min_median_max']); print('e2e', d['e2e']); print('roof', d['roofline']['frac'], d['roofline']['achieved']); print(d['stages_ms_per_projection']); print('clocks', d['clocks']); print('fp32', d['fp32']['value'])"
