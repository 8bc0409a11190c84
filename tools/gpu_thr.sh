for T in 1e-15 1e-14 1e-13; do
  echo "thr=$T"; PSD_JACOBI_THR=$T PSD_JACOBI_TIMERS=1 timeout 100 python tools/probe_eigh.py 272 2 2>&1 | tail -2
  PSD_JACOBI_THR=$T timeout 300 python bench.py --steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print(round(d['value'],2), d['stages_ms_per_projection']['eigh'], d['step_ms_min_median_max'])"
  PSD_JACOBI_THR=$T timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ozaki_syrk.py -m gpu -q -p no:cacheprovider -k "config3_shape or golden or rank_deficient or config2" 2>&1 | tail -1
done
