"""Repeat the C4-shape sharded-driver case (tests/test_gpu_parity.py::test_config4_shape_reduced_n)
to expose nondeterminism: every KernelOps call's output is checksummed and compared with the
first repetition's, so a divergence names the first kernel whose result changed.
usage: python tools/flaky_c4.py REPS [heat_seconds]"""
import hashlib, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402
from paper_2410_19208_b200 import workloads  # noqa: E402
from paper_2410_19208_b200.sharded import KernelOps, sharded_ran_proj  # noqa: E402
from oracle import psd_oracle as orc  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
heat = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0


def digest(v):
    if isinstance(v, torch.Tensor):
        return hashlib.sha1(v.detach().contiguous().cpu().numpy().tobytes()).hexdigest()[:12]
    if isinstance(v, (tuple, list)):
        return "|".join(digest(x) for x in v)
    return repr(v)


class Rec(KernelOps):
    def __init__(self, dev):
        super().__init__(dev)
        self.log = []

    def _wrap(name):
        def f(self, *a, **k):
            out = getattr(KernelOps, name)(self, *a, **k)
            self.log.append((name, digest(out)))
            return out
        return f

    for _n in ["xmul", "matmul", "gram", "chol_inv", "eigh", "scale_columns", "syrk_window", "max_abs"]:
        locals()[_n] = _wrap(_n)


n, k, p, q = 8192, 512, 32, 2
xd = workloads.c4_rows(n, 0, n, seed=5)
om = np.random.default_rng(6).standard_normal((n, k + p))
omd = torch.from_numpy(om).cuda()
ref = orc.ran_proj(xd.cpu().numpy(), k, p, q, omega=om).result
if heat > 0:   # warm the GPU up like the rest of the suite does
    a = torch.randn(8192, 8192, device="cuda")
    t0 = time.time()
    while time.time() - t0 < heat:
        a = (a @ a).clamp_(-1, 1)
    torch.cuda.synchronize()
first = None
for r in range(reps):
    ops = Rec("cuda")
    rep = sharded_ran_proj(xd, 0, n, omd, psd.RangeParams(k=k, l=p, q=q), ops=ops)
    res = rep.result_rows
    err = float(np.linalg.norm(res.cpu().numpy() - ref) / np.linalg.norm(ref))
    if first is None:
        first = ops.log
        print(f"rep 0: err {err:.2e}, {len(ops.log)} kernel calls", flush=True)
        continue
    bad = [(i, a[0]) for i, (a, b) in enumerate(zip(first, ops.log)) if a != b]
    print(f"rep {r}: err {err:.2e} first divergence {bad[:3] if bad else None}", flush=True)
