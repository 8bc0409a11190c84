# FP32 prefetch: tests + FP32 leg with and without the pipelined batch
timeout 900 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_fp32.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in "" "--no-prefetch"; do
timeout 600 python bench.py --steps 16 --warmup 3 --no-c4 --no-e2e --no-cpu-baseline --no-scaled --no-peaks $v 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); f=d['fp32']; print('$v', 'fp64', round(d['value'],2), 'fp32', round(f['value'],2), f['step_ms_min_median_max'], f['stages_ms_per_projection'])"
done
