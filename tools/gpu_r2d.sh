# round 2: row maxima from the symmetry pass → single-pass residues; validation inside psd_ran_proj
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pt_r2d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2d.log
F="--steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $F > gpurun_out/b_r2d.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"residues_rows|sym_stats" -c 6 --csv python bench.py --steps 1 --warmup 1 --pool 1 --no-fp32 --no-scaled --no-c4 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r2d.csv 2>&1
tail -3 gpurun_out/pt_r2d.log
