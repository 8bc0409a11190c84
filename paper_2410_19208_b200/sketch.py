"""Randomized range finder, power iteration and the min-eigenvalue shift trick
on the GPU (mirrors psdcone/sketch.py)."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, errors
from ._tensors import DeviceRng, as_device, draw_gaussian, require_square

RANK_TRUNCATION_FACTOR = 1e-12  # sketch.py:12


@dataclass(frozen=True)
class RangeParams:
    """sketch.py:15-39: target rank k, oversampling l, power exponent q."""

    k: int
    l: int = 10
    q: int = 0
    seed: int | None = None

    def __post_init__(self):
        if self.k < 1:
            raise errors.error("InvalidParams", f"target rank k must be >= 1, got {self.k}")
        if self.l < 0:
            raise errors.error("InvalidParams", f"oversampling l must be >= 0, got {self.l}")
        if self.q < 0:
            raise errors.error("InvalidParams", f"power exponent q must be >= 0, got {self.q}")

    @property
    def width(self):
        return self.k + self.l


def orthonormality_defect(q):
    """sketch.py:42-46: ‖QᵀQ − I‖_F."""
    if isinstance(q, torch.Tensor):
        q = q.to(torch.float64)
        return float(torch.linalg.matrix_norm(q.T @ q - torch.eye(q.shape[1], dtype=q.dtype,
                                                                     device=q.device)).item())
    q = np.asarray(q, dtype=float)
    return float(np.linalg.norm(q.T @ q - np.eye(q.shape[1])))


def _omega(omega, rng, n, width, device):
    if omega is not None:
        om = as_device(omega, device).t
        if tuple(om.shape) != (n, width):
            raise errors.error("DimensionMismatch", f"omega has shape {tuple(om.shape)}, expected {(n, width)}")
        return om
    return draw_gaussian(rng, (n, width), device)


def range_finder(x, params, rng, strict=False, *, omega=None):
    """sketch.py:53-93 on the GPU: (XXᵀ)^q XΩ with q ≥ 2 re-orthonormalisation,
    truncated economy QR (columns with |R_ii| ≤ 1e-12‖Y‖_F dropped)."""
    op = as_device(x)
    t = op.t
    if t.dim() != 2:
        raise errors.error("InvalidParams", f"expected a matrix, got shape {tuple(t.shape)}")
    m, n = int(t.shape[0]), int(t.shape[1])
    width = params.width
    if width > min(m, n):
        raise errors.error("InvalidParams", f"k+l = {width} exceeds min(m, n) = {min(m, n)}")
    om = _omega(omega, rng, n, width, op.device)
    lib = _native.load_library()
    plan = _native.get_plan(max(m, n), width, op.device)
    basis = torch.empty((m, width), dtype=torch.float64, device=op.device)
    wout = ctypes.c_int32(0)
    flags = _native.FLAG_STRICT if strict else 0
    _native.check(lib.psd_range_finder(plan.handle, _native.ptr(t), m, n, n, _native.ptr(om),
                                       om.stride(0), width, params.q, 0.0, flags,
                                       _native.ptr(basis), width, ctypes.byref(wout),
                                       _native.stream_handle(op.device)))
    return op.give_back(basis[:, : wout.value].contiguous())


def _power_iteration_device(op, n_iter, v0, shift=0.0):
    n = require_square(op)
    lib = _native.load_library()
    plan = _native.get_plan(n, 1, op.device)
    res = ctypes.c_double(0.0)
    _native.check(lib.psd_power_iteration(plan.handle, _native.ptr(op.t), n, n, float(shift),
                                          _native.ptr(v0), int(n_iter), ctypes.byref(res),
                                          _native.stream_handle(op.device)))
    return res.value


def power_iteration(x, n_iter, rng, *, v0=None):
    """sketch.py:96-114: exactly n_iter normalised GEMVs from a Gaussian start."""
    op = as_device(x)
    if n_iter < 1:
        raise errors.error("InvalidParams", f"power iteration needs n_iter >= 1, got {n_iter}")
    n = int(op.t.shape[0])
    v = as_device(v0, op.device).t if v0 is not None else draw_gaussian(rng, n, op.device)
    return _power_iteration_device(op, n_iter, v)


def min_eig_magnitude_device(op, n_iter, rng, v1=None, v2=None, bitwise_symmetric=False):
    """``bitwise_symmetric``: the caller verified X == Xᵀ exactly (project() runs
    require_symmetric first, projection.py:189), so the 2(N+1) products read only X's lower
    triangle (psd_min_eig_magnitude_ex, half the HBM traffic)."""
    n = require_square(op)
    if n_iter < 1:
        raise errors.error("InvalidParams", f"power iteration needs n_iter >= 1, got {n_iter}")
    a = as_device(v1, op.device).t if v1 is not None else draw_gaussian(rng, n, op.device)
    b = as_device(v2, op.device).t if v2 is not None else draw_gaussian(rng, n, op.device)
    lib = _native.load_library()
    plan = _native.get_plan(n, 1, op.device)
    res = ctypes.c_double(0.0)
    flags = _native.FLAG_ASSUME_SYMMETRIC if bitwise_symmetric else 0
    _native.check(lib.psd_min_eig_magnitude_ex(plan.handle, _native.ptr(op.t), n, n, _native.ptr(a),
                                               _native.ptr(b), int(n_iter), flags, ctypes.byref(res),
                                               _native.stream_handle(op.device)))   # sketch.py:126-129
    return res.value


def min_eig_magnitude(x, n_iter, rng, *, v1=None, v2=None):
    """sketch.py:117-129 (Alg. 5): |σ₁ − PI(X − σ₁I)| (the shift is fused, not materialised)."""
    return min_eig_magnitude_device(as_device(x), n_iter, rng, v1, v2)


__all__ = ["RangeParams", "orthonormality_defect", "range_finder", "power_iteration",
           "min_eig_magnitude", "DeviceRng", "RANK_TRUNCATION_FACTOR"]
