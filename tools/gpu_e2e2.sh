cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 600 python tools/probe_e2e.py 2>&1 | tail -1; done
timeout 900 python bench.py --no-fp32 --no-cpu-baseline --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench value', d['value'], 'e2e', d['e2e']['value'])"
