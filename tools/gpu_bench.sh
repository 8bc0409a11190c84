cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.log
timeout 300 python tools/profile_gemm.py 32768 272 5 nn > gpurun_out/gemm_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -s 2 -c 1 -o gpurun_out/gemm_full -f python tools/profile_gemm.py 32768 272 4 nn > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
cat gpurun_out/gemm_plain.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ls -la gpurun_out
