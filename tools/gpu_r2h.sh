# round 2: row maxima folded into the symmetry compute loop; SYRK capture after the MMA-loop fix
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_r2h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2h.log
F="--steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled"
timeout 300 python bench.py $F > gpurun_out/b_r2h.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"sym_stats" -c 2 --csv python bench.py --steps 1 --warmup 1 --pool 1 --no-fp32 --no-scaled --no-c4 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r2h.csv 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:i8_syrk -c 1 -o gpurun_out/syrk_r2h python tools/probe_syrk.py 32768 158 1 > gpurun_out/syrk_ncu_h.log 2>&1
tail -3 gpurun_out/pt_r2h.log
