"""Full-size BASELINE config 3 parity (n = 32768, k = 256, p = 16, q = 1): the GPU
FP64 path (INT8 engine products + INT8 reconstruction) against the CPU oracle
(the reference's numpy/LAPACK calls, oracle/psd_oracle.py) on the identical X
and Ω.  Needs ≈40 GB of host RAM and a few minutes of the host's cores.

    python tools/parity_c3_full.py [seed]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402
from oracle import psd_oracle as orc  # noqa: E402


def main():
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    n, k, p, q = 32768, 256, 16, 1
    dev = torch.device("cuda", 0)
    xd = psd.workloads.c3_device(n, seed=seed, device=dev)
    om = np.random.default_rng(seed + 100).standard_normal((n, k + p))
    t0 = time.perf_counter()
    rep = psd.ran_proj(xd, psd.RangeParams(k=k, l=p, q=q), None, omega=torch.from_numpy(om).to(dev))
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    res = rep.result.cpu().numpy()
    x = xd.cpu().numpy()
    del xd
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    o = orc.ran_proj(x, k, p, q, omega=om)
    t_cpu = time.perf_counter() - t0
    err = np.linalg.norm(res - o.result) / np.linalg.norm(o.result)
    print(f"C3 full size n={n} k={k} p={p} q={q} seed={seed}: rel Frobenius {err:.3e} (bar 1e-10); "
          f"rank {rep.effective_rank}/{o.effective_rank}, width {rep.basis_width}/{o.basis_width}, "
          f"engines {rep.device_info['sketch_engine']}/{rep.device_info['recon_engine']}, "
          f"bitwise symmetric {np.array_equal(res[:2048, :2048], res[:2048, :2048].T)}; "
          f"GPU call {t_gpu:.2f} s (incl. first-call setup), CPU oracle {t_cpu:.1f} s on {os.cpu_count()} cores",
          flush=True)


if __name__ == "__main__":
    main()
