# round 2: Jacobi with 64x64 subproblems (JB = 32) from m >= 160
for JB in 16 32; do echo "JB=$JB"; PSD_JACOBI_JB=$JB PSD_JACOBI_TIMERS=1 timeout 120 python tools/probe_eigh.py 272 3 2>&1 | tail -2; PSD_JACOBI_JB=$JB timeout 120 python tools/probe_eigh.py 544 2 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_r2l.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2l.log
F="--steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled"
timeout 300 python bench.py $F > gpurun_out/b_r2l.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b_r2l.json').read().strip().split(chr(10))[-1]); print(round(d['value'],2), d['stages_ms_per_projection'])"
tail -3 gpurun_out/pt_r2l.log
