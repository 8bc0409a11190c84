# deferred final-QR passes: GPU suite (quick) + C1/C2/C3 lines, deferred vs not (PSD_QR_DEFER=0)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not full_size" 2>&1 | tail -1
for rep in 1 2; do for v in 1 0; do for C in c1 c2; do PSD_QR_DEFER=$v timeout 300 python bench.py --config $C --steps 30 --warmup 3 --no-e2e --no-peaks --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('defer=$v $C', round(d['value'],1), d.get('stages_ms_per_projection',{}).get('qr'))"; done; done; done
