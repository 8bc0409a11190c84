# round 2: SYRK with 16 epilogue warps (1 column group each)
timeout 900 python -m pytest tests/test_gpu_ozaki_syrk.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_r2i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2i.log
timeout 120 python tools/probe_syrk.py 32768 158 5 > gpurun_out/syrk_r2i.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"i8_syrk" -c 3 --csv python tools/probe_syrk.py 32768 158 3 > gpurun_out/ncu_r2i.csv 2>&1
F="--steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled"
timeout 300 python bench.py $F > gpurun_out/b_r2i.json 2>&1
tail -3 gpurun_out/pt_r2i.log
