# A/B of the pipelined batch (psd_plan_prefetch) variants at C3: bench line summary per variant
F="--steps 16 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled --no-peaks"
run() { tag=$1; shift; env "$@" timeout 300 python bench.py $F > gpurun_out/b_$tag.json 2>gpurun_out/b_$tag.err; python -c "import json; d=json.loads(open('gpurun_out/b_$tag.json').read().strip().split(chr(10))[-1]); s=d['stages_ms_per_projection']; print('$tag', round(d['value'],2), round(d['ms_per_step'],2), [round(v,1) for v in d['step_ms_min_median_max']], {k: round(v,2) for k,v in s.items()}, d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for rep in 1 2; do
run off$rep PSD_PREFETCH=0
run qr$rep PSD_PREFETCH=1
done
