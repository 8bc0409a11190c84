cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c3 c2 c1; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; tail -2 gpurun_out/bench_$c.err
done
timeout 900 python bench.py --config c5 --steps 300 --warmup 3 > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"; tail -3 gpurun_out/bench_c5.err
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.log 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"; tail -3 gpurun_out/bench_c4.err
for c in c3 c2 c1 c5 c4; do echo "== $c"; cut -c1-1500 gpurun_out/bench_$c.log; done
