# quick GPU validation: the -m gpu suite without the two full-size C3 cases, then a short C3 bench
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_quick.log
F="--steps 16 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled --no-peaks"
for pf in 1 0; do
PSD_PREFETCH=$pf timeout 300 python bench.py $F > gpurun_out/b_quick$pf.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b_quick$pf.json').read().strip().split(chr(10))[-1]); print('prefetch=$pf', round(d['value'],2), d['ms_per_step'], d['stages_ms_per_projection'])"
done
tail -2 gpurun_out/pt_quick.log
