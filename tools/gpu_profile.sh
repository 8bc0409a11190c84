cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# dominant kernel: TMA DMMA GEMM at C3 shape, full ncu set on one launch
timeout 300 python tools/profile_gemm.py 32768 272 4 nn > gpurun_out/gemm_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tma_kernel -s 2 -c 1 -o gpurun_out/gemm_tma_full -f python tools/profile_gemm.py 32768 272 4 nn > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
# launch list of the bench command (short)
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
cat gpurun_out/gemm_plain.log; tail -2 gpurun_out/bench_small.log | cut -c1-300
