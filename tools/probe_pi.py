"""HBM roofline check of the power-iteration GEMV path at C3 size."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2410_19208_b200 as psd
from paper_2410_19208_b200 import workloads
dev = torch.device("cuda", 0)
n = 32768
x = workloads.c3_device(n, seed=3, device=dev)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    v = psd.power_iteration(x, 10, np.random.default_rng(1))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    gb = 11 * 8 * n * n / 1e9
    print(f"power_iteration N=10: {dt*1e3:.2f} ms, {gb/dt:.0f} GB/s of X reads, value {v:.6f}")
for it in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    v = psd.min_eig_magnitude(x, 10, np.random.default_rng(1))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    gb = 22 * 8 * n * n / 1e9
    print(f"min_eig_magnitude N=10: {dt*1e3:.2f} ms, {gb/dt:.0f} GB/s, value {v:.6f}")
