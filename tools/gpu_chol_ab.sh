# A/B of the CholeskyQR factor kernel's CTA size (PSD_CHOL_NT=256|512): phase cycles, then C1/C2/C3 bench lines
for NT in 256 512; do echo "== NT=$NT"; PSD_CHOL_NT=$NT PSD_CHOL_TIMERS=1 timeout 300 python tools/probe_chol.py 8192 256 2>&1 | tail -2; PSD_CHOL_NT=$NT PSD_CHOL_TIMERS=1 timeout 300 python tools/probe_chol.py 8192 128 2>&1 | tail -1; done
F="--steps 20 --warmup 3 --no-fp32 --no-c4 --no-e2e --no-cpu-baseline --no-scaled --no-peaks"
for rep in 1 2 3; do for NT in 256 512; do for C in c1 c2 c3; do
  PSD_CHOL_NT=$NT timeout 300 python bench.py --config $C $F 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('NT=$NT $C', round(d['value'],2), round(d['ms_per_step'],3), 'qr', d['stages_ms_per_projection']['qr'], d['clocks']['sm_mhz'])"
done; done; done
