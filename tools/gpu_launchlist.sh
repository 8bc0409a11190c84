# ncu launch list (per-kernel durations, serialized, cold) of projections: bash tools/gpu_launchlist.sh [config]
C=${1:-c3}
O=gpurun_out/ll; mkdir -p $O
F="--config $C --steps 2 --warmup 1 --pool 1 --no-peaks --no-fp32 --no-scaled --no-e2e --no-cpu-baseline --no-c4 --no-prefetch"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip ${SKIP:-0} -c 2000 --csv --log-file $O/launches_$C.csv python bench.py $F > $O/ncu_list_$C.log 2>&1
echo rc=$?
