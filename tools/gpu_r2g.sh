# round 2: leaner SYRK MMA/producer loops; symmetry pass with row maxima (row-major vs diagonal order)
timeout 900 python -m pytest tests/test_gpu_ozaki_syrk.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_r2g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2g.log
timeout 120 python tools/probe_syrk.py 32768 158 5 > gpurun_out/syrk_r2g.log 2>&1
F="--steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled"
timeout 300 python bench.py $F > gpurun_out/b_r2g.json 2>&1
PSD_SYM_ORDER=diag timeout 300 python bench.py $F > gpurun_out/b_r2g_diag.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"sym_stats|i8_syrk" -c 4 --csv python bench.py --steps 1 --warmup 1 --pool 1 --no-fp32 --no-scaled --no-c4 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r2g.csv 2>&1
tail -3 gpurun_out/pt_r2g.log
