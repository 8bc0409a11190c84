"""Repeat the C3-shape parity case to expose nondeterminism; on a bad rep,
report which stage diverged (eigenvalues of T vs oracle, rank, QR passes)."""
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
dref = np.sort(ref.factors[1])
bad = 0
first = None
for i in range(reps):
    rep = psd.ran_proj(x, psd.RangeParams(k=256, l=16, q=1), None, omega=om, return_factors=True)
    e = float(np.linalg.norm(rep.result - ref.result) / np.linalg.norm(ref.result))
    if first is None:
        first = rep.result.copy()
    drift = float(np.abs(rep.result - first).max())
    if e > 1e-10:
        bad += 1
        d = np.sort(rep.factors[1])
        de = float(np.abs(d - dref).max() / np.abs(dref).max()) if d.size == dref.size else -1
        print(f"BAD rep {i}: err {e:.2e} eigval-dev {de:.2e} info {rep.device_info}", flush=True)
    elif drift > 0:
        print(f"rep {i}: ok err {e:.2e} but differs from rep 0 by {drift:.2e}", flush=True)
print("BAD", bad, "of", reps)
