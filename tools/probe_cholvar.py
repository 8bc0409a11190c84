"""Residual of the CholeskyQR factor kernel (psd_chol_inv) on graded SPD matrices, for A/B of kernel
variants (PSD_CHOL_NT, PSD_CHOL_PIVOT): ‖LLᵀ − G‖/‖G‖, ‖L − L_ref‖/‖L_ref‖ (torch.linalg.cholesky), ‖RinvᵀLᵀ... − I‖."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402
from paper_2410_19208_b200.sharded import KernelOps  # noqa: E402
ops = KernelOps("cuda")
g0 = torch.Generator(device="cuda").manual_seed(3)
for m in (50, 144, 272, 544):
    for kappa in (1e2, 1e6, 1e10):
        y = torch.randn(4096, m, dtype=torch.float64, device="cuda", generator=g0)
        q = torch.linalg.qr(y)[0]
        s = torch.logspace(0, -torch.log10(torch.tensor(kappa)).item() / 2, m, dtype=torch.float64, device="cuda")
        v = torch.linalg.qr(torch.randn(m, m, dtype=torch.float64, device="cuda", generator=g0))[0]
        a = (q * s) @ v.T
        g = a.T @ a
        g = (g + g.T) / 2
        l_, rinv, info, trace, dmin, dmax = ops.chol_inv(g.clone(), 0.0)
        torch.cuda.synchronize()
        lref = torch.linalg.cholesky(g)
        res = ((l_ @ l_.T - g).norm() / g.norm()).item()
        dl = ((l_ - lref).norm() / lref.norm()).item()
        inv = ((rinv.T @ l_ - torch.eye(m, dtype=torch.float64, device="cuda")).abs().max()).item()
        print(f"m={m} kappa(G)={kappa:.0e} info={info} resid {res:.2e} dL {dl:.2e} |RinvT L - I| {inv:.2e} "
              f"ref resid {((lref @ lref.T - g).norm() / g.norm()).item():.2e}", flush=True)
