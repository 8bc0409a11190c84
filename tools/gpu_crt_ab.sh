# CRT variants: correctness (INT8-engine tests) and per-launch durations (ncu launch list)
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
F="--steps 1 --warmup 1 --pool 1 --no-peaks --no-fp32 --no-scaled --no-e2e --no-cpu-baseline --no-c4 --no-prefetch"
for v in table float; do
PSD_OZ_CRT=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:crt --csv --log-file gpurun_out/crt_$v.csv python bench.py $F > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/crt_$v.csv')))
h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
ki=rows[h].index('Kernel Name'); vi=rows[h].index('Metric Value')
v=[(r[ki][:30], float(r[vi].replace(',',''))/1000) for r in rows[h+1:] if len(r)>vi]
big=[t for k,t in v if t > 60]
print('$v', 'n', len(v), 'big avg us', round(sum(big)/max(len(big),1),1), 'small', [round(t,1) for k,t in v if t<=60][:4])
PY
done
