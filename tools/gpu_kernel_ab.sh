# usage: bash tools/gpu_kernel_ab.sh <kernel regex> <ENV=value for variant B> [pytest files...]
# per-launch durations (ncu launch list, one C3 step) of the matching kernels, default vs variant B
K=$1; V=$2; shift 2
[ $# -gt 0 ] && timeout 900 python -m pytest "$@" -x -q -p no:cacheprovider 2>&1 | tail -1
F="--steps 1 --warmup 1 --pool 1 --no-peaks --no-fp32 --no-scaled --no-e2e --no-cpu-baseline --no-c4 --no-prefetch"
for tag in default variant; do
  if [ $tag = variant ]; then E="$V"; else E="PSD_NONE=1"; fi
  env $E timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$K --csv --log-file gpurun_out/kab_$tag.csv python bench.py $F > /dev/null 2>&1
  python - <<PY
import csv, collections
rows=list(csv.reader(open('gpurun_out/kab_$tag.csv')))
h=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
ki=rows[h].index('Kernel Name'); vi=rows[h].index('Metric Value')
d=collections.defaultdict(list)
for r in rows[h+1:]:
    if len(r)>vi: d[r[ki].split('(')[0][-40:]].append(float(r[vi].replace(',',''))/1000)
print('$tag', {k: (len(v), round(sum(v)/len(v),1)) for k,v in d.items()})
PY
done
