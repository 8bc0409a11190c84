# Round-end evidence on one B200: GPU suite, smoke, bench (all legs), other configs,
# the reference arm at full size, the ncu launch list and full captures of the top kernels.
set -x
O=gpurun_out/ev
mkdir -p $O
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 16 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
for C in c1 c2; do timeout 600 python bench.py --config $C --steps 20 --warmup 3 --no-e2e >> $O/bench_configs.jsonl 2>> $O/bench_configs.err; done
timeout 900 python bench.py --config c5 --steps 300 --warmup 3 >> $O/bench_configs.jsonl 2>> $O/bench_configs.err
timeout 600 python bench.py --config c4 --c4-steps 3 >> $O/bench_configs.jsonl 2>> $O/bench_configs.err
timeout 1500 python bench.py --impl reference --steps 16 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
F="--steps 2 --warmup 1 --pool 1 --no-peaks --no-fp32 --no-scaled --no-e2e --no-cpu-baseline --no-c4"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 450 -c 1500 --csv --log-file $O/launches_bench.csv python bench.py $F --no-prefetch > $O/ncu_list.log 2>&1
timeout 600 python tools/selfcheck.py 10 > $O/selfcheck.log 2>&1
for K in i8_gemm2 residues_rows_max i8_syrk sym_stats symv_tiles tc32_gemm2 jacobi_persistent crt1_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o $O/full_$K python bench.py --steps 1 --warmup 1 --pool 1 --no-peaks --no-e2e --no-cpu-baseline --no-c4 > $O/ncu_full_$K.log 2>&1
done
tail -n 3 $O/pytest_gpu.log $O/smoke.log $O/selfcheck.log
