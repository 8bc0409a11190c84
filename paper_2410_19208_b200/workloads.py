"""Seeded synthetic inputs of BASELINE.json's configs, generated directly in
HBM (torch is only the data generator here; nothing below is timed).

C3 (BASELINE.json configs[2]): X = U diag(s) Uᵀ − W diag(t) Wᵀ + 1e-3·E with
U, W (n×200) orthonormal, s = geomspace(1e3, 1, 200), t ~ U[0, 10], E a
symmetric Wigner matrix, explicitly symmetrised (bitwise) afterwards.
"""

from __future__ import annotations

import math

import torch

from . import _native


def _symmetrize_inplace(x):
    lib = _native.load_library()
    _native.check(lib.psd_symmetrize(_native.ptr(x), x.shape[0], x.stride(0),
                                     _native.stream_handle(x.device)))


def wigner_device(n, seed=0, device="cuda", out=None):
    """(G + Gᵀ)/(2√n), bitwise symmetric."""
    g = torch.Generator(device=device).manual_seed(int(seed))
    x = out if out is not None else torch.empty((n, n), dtype=torch.float64, device=device)
    x.normal_(generator=g)
    _symmetrize_inplace(x)          # (G + Gᵀ)/2
    x.mul_(1.0 / math.sqrt(n))      # → (G + Gᵀ)/(2√n)
    return x


def c3_device(n, seed=0, rank=200, device="cuda", out=None):
    g = torch.Generator(device=device).manual_seed(int(seed) + 7919)
    x = wigner_device(n, seed, device, out)
    x.mul_(1e-3)
    u = torch.linalg.qr(torch.randn(n, rank, dtype=torch.float64, device=device, generator=g))[0]
    w = torch.linalg.qr(torch.randn(n, rank, dtype=torch.float64, device=device, generator=g))[0]
    s = torch.logspace(3.0, 0.0, rank, dtype=torch.float64, device=device)
    t = 10.0 * torch.rand(rank, dtype=torch.float64, device=device, generator=g)
    x.addmm_(u * s, u.T)
    x.addmm_(w * (-t), w.T)
    _symmetrize_inplace(x)
    return x


def c1_device(n=1000, seed=0, device="cuda"):
    """Config 1: Haar V, λ₁..₃₀ = geomspace(1e2, 1e-2, 30), rest U[−1, 0]."""
    g = torch.Generator(device=device).manual_seed(int(seed))
    v = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=device, generator=g))[0]
    lam = torch.cat([torch.logspace(2.0, -2.0, 30, dtype=torch.float64, device=device),
                     -torch.rand(n - 30, dtype=torch.float64, device=device, generator=g)])
    x = (v * lam) @ v.T
    _symmetrize_inplace(x)
    return x
