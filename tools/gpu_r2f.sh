# round 2: diagonal-major symmetry pass; SYRK full ncu capture
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_r2f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2f.log
F="--steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled"
timeout 300 python bench.py $F > gpurun_out/b_r2f.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"residues_rows|sym_stats" -c 4 --csv python bench.py --steps 1 --warmup 1 --pool 1 --no-fp32 --no-scaled --no-c4 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r2f.csv 2>&1
timeout 120 python tools/probe_syrk.py 32768 158 1 > gpurun_out/syrk_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:i8_syrk -c 1 -o gpurun_out/syrk_r2 python tools/probe_syrk.py 32768 158 1 > gpurun_out/syrk_ncu.log 2>&1
tail -3 gpurun_out/pt_r2f.log
