"""Symmetric-matrix core on the GPU (mirrors psdcone/symmetric.py).

Validation, the k×k eigensolver and the exact projection run in
libpsdproj.so; host-side pieces are only the reference's RNG plumbing
(``rng_from_seed`` / ``gaussian_matrix`` draw from numpy exactly as
symmetric.py:19-28 and :131-135 do, so Ω matches the reference bit-for-bit).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, errors
from ._tensors import DeviceRng, as_device, require_square

SYM_TOL_FACTOR = 1e-10  # symmetric.py:16


@dataclass(frozen=True)
class SymStats:
    max_abs: float
    defect: float
    bitwise: bool


def rng_from_seed(seed):
    """symmetric.py:19-28 (DeviceRng instances pass through too)."""
    if isinstance(seed, (np.random.Generator, DeviceRng)):
        return seed
    return np.random.default_rng(seed)


def gaussian_matrix(rows, cols, rng):
    """symmetric.py:131-135 — host numpy draw (the reference's stream)."""
    if rows < 1 or cols < 1:
        raise ValueError("gaussian_matrix requires rows, cols >= 1")
    return rng.standard_normal((rows, cols))


def check_symmetric_device(op, tol=None):
    """require_symmetric on a device operand → SymStats; raises like symmetric.py:53-56."""
    n = require_square(op)
    lib = _native.load_library()
    plan = _native.get_plan(n, 1, op.device)
    stats = (ctypes.c_double * 3)()
    st = lib.psd_require_symmetric(plan.handle, _native.ptr(op.t), n, n,
                                   -1.0 if tol is None else float(tol), stats,
                                   _native.stream_handle(op.device))
    _native.check(st)
    return SymStats(max_abs=stats[0], defect=stats[1], bitwise=stats[2] == 1.0)


def require_symmetric(a, tol=None):
    """symmetric.py:39-57: validate on the GPU, return ``a`` as float64."""
    op = as_device(a)
    check_symmetric_device(op, tol)
    if isinstance(a, torch.Tensor):
        return op.t if a.is_cuda else a.to(torch.float64)
    return np.asarray(a, dtype=float)


def symmetrize(a):
    """symmetric.py:31-36: (A + Aᵀ)/2 (computed by the library's mirror kernel)."""
    op = as_device(a)
    t = op.t
    if t.dim() != 2 or t.shape[0] != t.shape[1]:
        raise errors.error("NonSquareError", f"expected a square matrix, got shape {tuple(t.shape)}")
    out = t.clone()
    lib = _native.load_library()
    _native.check(lib.psd_symmetrize(_native.ptr(out), out.shape[0], out.shape[0],
                                     _native.stream_handle(op.device)))
    return op.give_back(out)


@dataclass(frozen=True)
class EigenDecomposition:
    """symmetric.py:60-65: X = U diag(values) Uᵀ, values descending."""

    values: object
    vectors: object


def eigh_device(op, validate=True):
    """(values, vectors) device tensors for a square device operand."""
    if validate:
        check_symmetric_device(op)
    m = require_square(op)
    lib = _native.load_library()
    plan = _native.get_plan(m, m, op.device)
    work = op.t.clone()
    vals = torch.empty(m, dtype=torch.float64, device=op.device)
    vecs = torch.empty((m, m), dtype=torch.float64, device=op.device)
    sweeps = ctypes.c_int32(0)
    _native.check(lib.psd_eigh(plan.handle, _native.ptr(work), m, m, _native.ptr(vals),
                               _native.ptr(vecs), m, ctypes.byref(sweeps),
                               _native.stream_handle(op.device)))
    return vals, vecs


def eigh(x):
    """symmetric.py:68-86: descending eigenvalues, largest-|entry| positive vectors."""
    op = as_device(x)
    vals, vecs = eigh_device(op)
    return EigenDecomposition(values=op.give_back(vals), vectors=op.give_back(vecs))


def reconstruct_device(w, d, n, device):
    """sym(W diag(d) Wᵀ) on the tensor cores (projection.py:72-78)."""
    r = int(d.numel())
    lib = _native.load_library()
    plan = _native.get_plan(n, max(r, 1), device)
    out = torch.empty((n, n), dtype=torch.float64, device=device)
    w = w.contiguous()
    _native.check(lib.psd_reconstruct(plan.handle, _native.ptr(w), n, w.stride(0) if r else 1,
                                      _native.ptr(d.contiguous()), r, _native.ptr(out), n,
                                      _native.stream_handle(device)))
    return out


def exact_psd_projection_device(op, validate=True):
    vals, vecs = eigh_device(op, validate)
    keep = vals > 0.0
    r = int(keep.sum().item())
    return reconstruct_device(vecs[:, :r], vals[:r], op.t.shape[0], op.device), vals, vecs, r


def exact_psd_projection(x):
    """symmetric.py:109-114: eigen-decompose and clip negative eigenvalues."""
    op = as_device(x)
    return op.give_back(exact_psd_projection_device(op)[0])


def frobenius_norm(x):
    """symmetric.py:89-91."""
    if isinstance(x, torch.Tensor):
        return float(torch.linalg.vector_norm(x.to(torch.float64)).item())
    return float(np.linalg.norm(np.asarray(x, dtype=float)))
