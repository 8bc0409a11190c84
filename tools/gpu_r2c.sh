# round 2: paired-moduli residue kernel — correctness + stage timing + ncu launch times
timeout 600 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_ozaki_syrk.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_r2c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2c.log
F="--steps 8 --warmup 3 --no-fp32 --no-scaled --no-c4 --no-e2e --no-cpu-baseline"
PSD_OZ_RES=limb timeout 300 python bench.py $F > gpurun_out/b_limb.json 2>&1
timeout 300 python bench.py $F > gpurun_out/b_dp.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:residues_rows -c 4 --csv python bench.py --steps 1 --warmup 1 --pool 1 --no-fp32 --no-scaled --no-c4 --no-e2e --no-cpu-baseline > gpurun_out/ncu_res_dp.csv 2>&1
PSD_OZ_RES=limb timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:residues_rows -c 4 --csv python bench.py --steps 1 --warmup 1 --pool 1 --no-fp32 --no-scaled --no-c4 --no-e2e --no-cpu-baseline > gpurun_out/ncu_res_limb.csv 2>&1
tail -3 gpurun_out/pt_r2c.log
