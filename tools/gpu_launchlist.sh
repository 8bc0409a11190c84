# ncu launch list (per-kernel durations, serialized, cold) of C3 projections
O=gpurun_out/ll; mkdir -p $O
F="--steps 2 --warmup 1 --pool 1 --no-peaks --no-fp32 --no-scaled --no-e2e --no-cpu-baseline --no-c4 --no-prefetch"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 450 -c 1500 --csv --log-file $O/launches.csv python bench.py $F > $O/ncu_list.log 2>&1
echo rc=$?
