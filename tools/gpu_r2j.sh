# round 2: deferred symmetry verdict (no stream drain before the first product)
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pt_r2j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_r2j.log
F="--steps 8 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled"
timeout 300 python bench.py $F > gpurun_out/b_r2j.json 2>&1
tail -3 gpurun_out/pt_r2j.log
