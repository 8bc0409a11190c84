# round 2: REDUX row maxima in the symmetry pass; Jacobi phase timers
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_r2e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2e.log
F="--steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled"
timeout 300 python bench.py $F > gpurun_out/b_r2e.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"residues_rows|sym_stats" -c 4 --csv python bench.py --steps 1 --warmup 1 --pool 1 --no-fp32 --no-scaled --no-c4 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r2e.csv 2>&1
PSD_JACOBI_TIMERS=1 timeout 120 python tools/probe_eigh.py 272 4 > gpurun_out/eigh_timers.log 2>&1
tail -3 gpurun_out/pt_r2e.log
