# A/B of the side-stream residue kernel's CTA size in the pipelined batch (PSD_PF_THREADS, PSD_PF_ROWS) at C3
F="--steps 16 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled --no-peaks"
run() { tag=$1; shift; env "$@" timeout 300 python bench.py $F > gpurun_out/b_$tag.json 2>gpurun_out/b_$tag.err; python -c "import json; d=json.loads(open('gpurun_out/b_$tag.json').read().strip().split(chr(10))[-1]); s=d['stages_ms_per_projection']; print('$tag', round(d['value'],2), round(d['ms_per_step'],2), [round(v,1) for v in d['step_ms_min_median_max']], {k: round(v,2) for k,v in s.items()}, d['clocks']['sm_mhz'], 'unpipelined', round(d['unpipelined']['value'],2))" 2>&1 | tail -1; }
for rep in 1 2 3; do
run t256_$rep PSD_PF_THREADS=256
run t128_$rep PSD_PF_THREADS=128
run t128r1_$rep PSD_PF_THREADS=128 PSD_PF_ROWS=1
run t64_$rep PSD_PF_THREADS=64 PSD_PF_ROWS=1
done
