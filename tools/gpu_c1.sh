cd $GRAFT_REPO_ROOT
for eng in int8 dmma int8 dmma; do
python bench.py --config c1 --fp64-engine $eng --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', '$eng', round(d['value'],1), d['step_ms_min_median_max'])"
done
for n in 2048 4096; do for eng in int8 dmma; do
python bench.py --config c2 --n $n --fp64-engine $eng --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 n=$n', '$eng', round(d['value'],1), d['step_ms_min_median_max'])"
done; done
