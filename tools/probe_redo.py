"""Launch counts of the q = 2 graded-spectrum case (tests/test_gpu_kernels.py::test_power_step_qr_redo_path):
a device-decided power-step QR that raises its flag shows up as a redo (more launches)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_19208_b200 as psd  # noqa: E402
n, k, l, q = 512, 24, 8, 2
g = np.random.default_rng(11)
u, _ = np.linalg.qr(g.standard_normal((n, n)))
lam = np.concatenate([np.geomspace(1e4, 1e-4, 20), -np.geomspace(1e2, 1e-3, 20), np.zeros(n - 40)])
x = (u * lam) @ u.T
x = (x + x.T) / 2
om = g.standard_normal((n, k + l))
rep = psd.ran_proj(x, psd.RangeParams(k=k, l=l, q=q), None, omega=om)
y = psd.ran_proj(psd.symmetric.symmetrize(np.eye(n) + 0.01 * (x + x.T)), psd.RangeParams(k=k, l=l, q=q), None, omega=om)
print("graded launches", rep.device_info["gpu_launches"], "well-conditioned launches", y.device_info["gpu_launches"])
