# launch lists of the small configs (C1, C2): per-kernel device time per projection
O=gpurun_out/ll; mkdir -p $O
for C in c1 c2; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/$C.csv python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-peaks > $O/$C.log 2>&1
python tools/launch_shares.py $O/$C.csv > $O/${C}_shares.txt 2>&1; head -25 $O/${C}_shares.txt
done
