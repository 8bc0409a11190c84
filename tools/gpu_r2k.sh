# round 2: Jacobi inner sweeps per subproblem solve (sweeps vs round cost)
for I in 1 2 3 4; do echo "inner=$I"; PSD_JACOBI_INNER=$I PSD_JACOBI_TIMERS=1 timeout 120 python tools/probe_eigh.py 272 3 2>&1 | tail -2; done
for I in 1 2 3; do PSD_JACOBI_INNER=$I timeout 300 python bench.py --steps 6 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('inner=$I', round(d['value'],2), d['stages_ms_per_projection']['eigh'])"; done
