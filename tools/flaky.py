"""Repeat the C3-shape n=4096 parity case to expose nondeterminism."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd
from oracle import psd_oracle as orc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
x = orc.c3_matrix(n, seed=7)
om = np.random.default_rng(8).standard_normal((n, 272))
ref = orc.ran_proj(x, 256, 16, 1, omega=om)
bad = 0
for i in range(reps):
    rep = psd.ran_proj(x, psd.RangeParams(k=256, l=16, q=1), None, omega=om)
    e = float(np.linalg.norm(rep.result - ref.result) / np.linalg.norm(ref.result))
    if e > 1e-10:
        bad += 1
    print(f"rep {i}: err {e:.2e} sweeps {rep.device_info['eig_sweeps']} rank {rep.effective_rank}", flush=True)
print("BAD", bad)
