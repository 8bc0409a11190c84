# symmetric α estimate: tests + the scaled bench leg
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_dropin.py -q -p no:cacheprovider -k "not full_size" 2>&1 | tail -2
timeout 600 python bench.py --steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-peaks 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); s=d['scaled']; print('c3', round(d['value'],2), 'scaled', round(s['value'],2), s['ms_per_step'], {k: s[k] for k in s if 'gemv' in k or 'alpha' in k})"
