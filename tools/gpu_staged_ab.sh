# direct vs smem-staged mirrored stores of the DMMA SYRK (PSD_STAGED_EPI): C1 line, DMMA-engine C3 reconstruction
# stage, then the full GPU suite on the default (direct stores)
F="--steps 12 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled --no-peaks"
for S in 0 1; do
  PSD_STAGED_EPI=$S timeout 300 python bench.py --config c1 $F 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('STAGED=$S c1', round(d['value'],1), d['stages_ms_per_projection'])"
  PSD_STAGED_EPI=$S timeout 300 python bench.py --config c3 --fp64-engine dmma $F 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('STAGED=$S c3-dmma', round(d['value'],2), d['stages_ms_per_projection'])"
done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rf > gpurun_out/suite_direct.log 2>&1; echo "rc=$?" >> gpurun_out/suite_direct.log; tail -3 gpurun_out/suite_direct.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
