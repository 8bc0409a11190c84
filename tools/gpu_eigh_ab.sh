# device time per psd_eigh (CUDA events) and sweep count per m (tools/probe_eigh2.py)
python tools/probe_eigh2.py 20 32 50 74 96
PSD_JACOBI_CTA=0 python tools/probe_eigh2.py 20 32 50 74 96
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" 2>&1 | tail -1
timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-e2e --no-peaks --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('c1', round(d['value'],1), d['ms_per_step'], d.get('stages_ms_per_projection'))"
timeout 600 python bench.py --config c5 --steps 100 --warmup 3 --no-peaks --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('c5', round(d['value'],1), d['ms_per_step'])"
