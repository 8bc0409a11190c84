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


def c4_rows(n, r0, r1, seed=0, rank=200, device="cuda", chunk_rows=None):
    """Rows [r0, r1) of BASELINE config 4's X (same form as config 3) generated
    independently on each rank yet bitwise symmetric as a whole:
    X = mirror(lower([U·s, −W·t]·[U, W]ᵀ)) + 1e-3·E with E keyed on
    (seed, min(i,j), max(i,j)); U, W orthonormal n×rank from a seed shared by
    all ranks."""
    lib = _native.load_library()
    g = torch.Generator(device=device).manual_seed(int(seed) + 104729)
    u = torch.linalg.qr(torch.randn(n, rank, dtype=torch.float64, device=device, generator=g))[0]
    w = torch.linalg.qr(torch.randn(n, rank, dtype=torch.float64, device=device, generator=g))[0]
    s = torch.logspace(3.0, 0.0, rank, dtype=torch.float64, device=device)
    t = 10.0 * torch.rand(rank, dtype=torch.float64, device=device, generator=g)
    a = torch.cat([u * s, -(w * t)], 1).contiguous()
    b = torch.cat([u, w], 1).contiguous()
    x = torch.empty((r1 - r0, n), dtype=torch.float64, device=device)
    st = _native.stream_handle(torch.device(device))
    step = chunk_rows or (r1 - r0)
    for c0 in range(r0, r1, step):
        c1 = min(r1, c0 + step)
        view = x[c0 - r0:c1 - r0]
        _native.check(lib.psd_syrk_window(_native.ptr(a), a.stride(0), _native.ptr(b), b.stride(0),
                                          n, a.shape[1], c0, c1, _native.ptr(view), view.stride(0), st))
    _native.check(lib.psd_fill_sym_gaussian(_native.ptr(x), x.stride(0), r0, r1 - r0, n,
                                            int(seed) & 0xFFFFFFFFFFFFFFFF,
                                            1e-3 / math.sqrt(2.0 * n), 1.0, st))
    return x


def c5_problem(n=4096, m=20000, nnz_per=4, seed=0, rank=10):
    """BASELINE config 5 as a ``SparseSdlsProblem`` (host COO triplets; the
    solver uploads them): constraint i holds ``nnz_per`` seeded off-diagonal
    N(0,1) entries, each stored at (r, c) and (c, r); b = A(Z Zᵀ) with Z n×rank
    Gaussian; C = Wigner + 2I; ρ = 1.  The draw order (positions, values, Z, G)
    is the one tests/ pin against the CPU restatement."""
    import numpy as np

    from .sdls import SparseSdlsProblem
    rng = np.random.default_rng(seed)
    r = rng.integers(0, n, size=(m, nnz_per))
    c = rng.integers(0, n - 1, size=(m, nnz_per))
    c += c >= r                                            # skip the diagonal
    v = rng.standard_normal((m, nnz_per))
    z = rng.standard_normal((n, rank))
    g = rng.standard_normal((n, n))
    rows = np.stack([r, c], axis=-1).reshape(-1)           # (r, c) then its mirror
    cols = np.stack([c, r], axis=-1).reshape(-1)
    vals = np.repeat(v, 2, axis=1).reshape(-1)
    con = np.repeat(np.arange(m), 2 * nnz_per)
    cmat = (g + g.T) / (2.0 * math.sqrt(n)) + 2.0 * np.eye(n)
    x0 = z @ z.T
    b = np.zeros(m)
    np.add.at(b, con, vals * x0[rows, cols])               # bᵢ = ⟨Aᵢ, X₀⟩
    return SparseSdlsProblem(cmat, 1.0, con, rows, cols, vals, b)


def c5_step_size(problem, iters=50, seed=0):
    """β = 1/L, L = λ_max of the constraint Gram ⟨Aᵢ, Aⱼ⟩_F, by power iteration
    on v ↦ A(A*(v)) over the COO triplets (host, set-up only)."""
    import numpy as np
    n, m = problem.n, problem.m
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(m)
    v /= np.linalg.norm(v)
    lam = 0.0
    for _ in range(iters):
        adj = np.zeros((n, n))
        np.add.at(adj, (problem.rows, problem.cols), v[problem.con] * problem.vals)
        w = np.zeros(m)
        np.add.at(w, problem.con, problem.vals * adj[problem.rows, problem.cols])
        lam = float(np.linalg.norm(w))
        v = w / lam
    return 1.0 / lam
