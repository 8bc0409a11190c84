"""Repeat the device eigensolver on fixed matrices and compare every result bit for bit with the
first (dataflow races in the persistent Jacobi show up as rare differing repetitions).
usage: python tools/flaky_eigh.py REPS m [m ...]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402
from paper_2410_19208_b200._tensors import Operand  # noqa: E402
from paper_2410_19208_b200.symmetric import eigh_device  # noqa: E402

reps = int(sys.argv[1])
for m in [int(v) for v in sys.argv[2:]]:
    rng = np.random.default_rng(m)
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    lam = np.concatenate([np.geomspace(1e3, 1, m // 2), -10 * rng.random(m - m // 2)])
    a = torch.from_numpy((q * lam) @ q.T).cuda()
    a = (a + a.T) / 2
    v0, w0 = eigh_device(Operand(a.clone(), "torch_cuda", a.device), validate=False)
    bad = 0
    for r in range(reps):
        v, w = eigh_device(Operand(a.clone(), "torch_cuda", a.device), validate=False)
        if not (torch.equal(v, v0) and torch.equal(w, w0)):
            bad += 1
            if bad <= 3:
                print(f"m={m} rep {r}: differs: max |dvals| {float((v - v0).abs().max()):.2e} "
                      f"max |dvecs| {float((w - w0).abs().max()):.2e}", flush=True)
    print(f"m={m}: {bad} of {reps} repetitions differ", flush=True)
