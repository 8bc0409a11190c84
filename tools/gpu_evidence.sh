cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for c in c1 c2; do timeout 600 python bench.py --config $c --no-e2e > gpurun_out/bench_$c.json 2>/dev/null; echo "$c rc=$?"; done
timeout 900 python bench.py --config c5 --steps 300 > gpurun_out/bench_c5.json 2>/dev/null; echo "c5 rc=$?"
timeout 1200 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.json 2>/dev/null; echo "c4 rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>/dev/null; echo "ref rc=$?"
