# round-1 refresh of the non-headline configs (C1, C2, C5, C4 at N=1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for c in c1 c2; do timeout 600 python bench.py --config $c --no-e2e >> gpurun_out/configs.jsonl 2>gpurun_out/cfg_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --config c5 --steps 300 >> gpurun_out/configs.jsonl 2>gpurun_out/cfg_c5.err; echo "c5 rc=$?"
timeout 1500 python bench.py --config c4 --steps 2 --warmup 1 >> gpurun_out/configs.jsonl 2>gpurun_out/cfg_c4.err; echo "c4 rc=$?"
