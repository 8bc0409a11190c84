cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['fp32']['value'], d['fp32']['ms_per_step'], d['fp32']['step_ms_min_median_max'], d['fp32']['stages_ms_per_projection'])"
