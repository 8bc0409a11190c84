"""CholeskyQR factor-step anatomy: run a few C3-shaped projections with PSD_CHOL_TIMERS=1
(chol_blocked_kernel prints per-phase cycles) at reduced n (the w×w work does not depend on n)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402
from paper_2410_19208_b200 import workloads  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
k = int(sys.argv[2]) if len(sys.argv) > 2 else 256
x = workloads.c3_device(n, seed=1, device=torch.device("cuda:0"))
for _ in range(3):
    psd.ran_proj(x, psd.RangeParams(k=k, l=16, q=1), psd.DeviceRng(seed=2))
torch.cuda.synchronize()
