"""Time the device eigensolver (psd.eigh) on a C3-like 272x272 compressed matrix."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 272
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
rng = np.random.default_rng(0)
q, _ = np.linalg.qr(rng.standard_normal((m, m)))
lam = np.concatenate([np.geomspace(1e3, 1, m // 2), -10 * rng.random(m - m // 2)])
a = (q * lam) @ q.T
a = (a + a.T) / 2
t = torch.from_numpy(a).cuda()
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vals, vecs = psd.symmetric.eigh_device(psd._tensors.as_device(t), validate=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    err = np.abs(np.sort(vals.cpu().numpy()) - np.sort(lam)).max()
    print(f"eigh m={m}: {dt*1e3:.3f} ms  max eig err {err:.2e}", flush=True)
