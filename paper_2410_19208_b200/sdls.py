"""Dual gradient ascent for semidefinite least squares (Alg. 6) on the GPU —
drop-in for psdcone.sdls.solve (sdls.py:164-265) at BASELINE config-5 scale.

The reference stacks the m constraint matrices densely (sdls.py:44; 2.68 TB
at n=4096, m=20000).  Here constraints are sparse (COO with every stored
entry explicit) and every iteration runs on the device:

* dual assembly C/ρ + Σ yᵢAᵢ (sdls.py:83-89): copy + per-position fixed-order
  scatter (``psd_sdls_assemble``) — bitwise symmetric for symmetric Aᵢ;
* one randomized projection per iteration (sdls.py:235) through
  ``psd_ran_proj`` with ``result = NULL``: only the factors W, d are formed,
  the n×n X₊ is never materialised inside the loop;
* traces Tr(AᵢX₊) on the factored X₊ = sym((W·D)·Wᵀ) at the stored entries
  (``psd_sdls_traces``), gradient, ‖grad‖ and the ascent step
  (``psd_sdls_step``).

RNG draw order matches the reference: y₀ (if not given), then per iteration
the two α start vectors (scaled method, on refresh iterations), then Ω.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, errors
from ._tensors import DeviceRng, Operand, default_device, draw_gaussian
from .projection import ALPHA_TOL_FACTOR, ProjectorConfig
from .sketch import min_eig_magnitude_device
from .symmetric import exact_psd_projection_device, reconstruct_device, rng_from_seed


class SparseSdlsProblem:
    """(C, ρ, {(Aᵢ, bᵢ)}) with Aᵢ as COO triplets: entry t belongs to
    constraint con[t] and contributes vals[t] at (rows[t], cols[t])."""

    def __init__(self, c, rho, con, rows, cols, vals, b):
        self.c = np.asarray(c, dtype=float)
        if rho <= 0:
            raise errors.error("InvalidParams", f"rho must be positive, got {rho}")
        self.rho = float(rho)
        self.con = np.asarray(con, dtype=np.int64)
        self.rows = np.asarray(rows, dtype=np.int64)
        self.cols = np.asarray(cols, dtype=np.int64)
        self.vals = np.asarray(vals, dtype=float)
        self.b = np.asarray(b, dtype=float).ravel()

    @property
    def n(self):
        return self.c.shape[0]

    @property
    def m(self):
        return self.b.size

    @classmethod
    def from_reference(cls, problem):
        """From psdcone.SdlsProblem (dense a_stack, sdls.py:21-57)."""
        if isinstance(problem, cls):
            return problem
        if hasattr(problem, "con") and hasattr(problem, "vals"):
            return cls(problem.c, problem.rho, problem.con, problem.rows, problem.cols,
                       problem.vals, problem.b)
        a = np.asarray(problem.a_stack)
        con, rows, cols = np.nonzero(a)
        return cls(problem.c, problem.rho, con, rows, cols, a[con, rows, cols], problem.b)


@dataclass
class TrajectoryPoint:
    iteration: int
    grad_norm: float
    feasibility_residual: float


@dataclass
class SolveReport:
    """sdls.py:139-161."""

    x_solution: object
    y_final: np.ndarray
    iterations: int
    grad_norm_final: float
    feasibility_residual: float
    objective: float
    projection_method: str
    converged: bool
    wall_time: float
    trajectory: list | None = None
    y_trajectory: list | None = None
    exact_feasibility_residual: float | None = None


class _DeviceProblem:
    """Device-resident index structures of a SparseSdlsProblem."""

    def __init__(self, prob, device):
        n, m = prob.n, prob.m
        dev = device
        self.n, self.m, self.device = n, m, dev
        self.cr = torch.from_numpy(prob.c / prob.rho).to(dev)
        self.b = torch.from_numpy(prob.b).to(dev)
        flat = prob.rows * n + prob.cols
        order = np.lexsort((prob.con, flat))            # by position, then constraint
        fl = flat[order]
        starts = np.flatnonzero(np.r_[True, fl[1:] != fl[:-1]]) if fl.size else np.zeros(0, np.int64)
        self.npos = int(starts.size)
        ptr = np.r_[starts, fl.size].astype(np.int32)
        self.pos = torch.from_numpy(fl[starts].astype(np.int64)).to(dev)
        self.ptr = torch.from_numpy(ptr).to(dev)
        self.econ = torch.from_numpy(prob.con[order].astype(np.int32)).to(dev)
        self.evals = torch.from_numpy(prob.vals[order]).to(dev)
        corder = np.argsort(prob.con, kind="stable")     # by constraint, stored order kept
        cptr = np.searchsorted(prob.con[corder], np.arange(m + 1)).astype(np.int32)
        self.crow = torch.from_numpy(prob.rows[corder].astype(np.int32)).to(dev)
        self.ccol = torch.from_numpy(prob.cols[corder].astype(np.int32)).to(dev)
        self.cval = torch.from_numpy(prob.vals[corder]).to(dev)
        self.cptr = torch.from_numpy(cptr).to(dev)
        self.lib = _native.load_library()

    def assemble(self, y, out):
        _native.check(self.lib.psd_sdls_assemble(
            _native.ptr(self.cr), self.n, _native.ptr(self.pos), _native.ptr(self.ptr),
            _native.ptr(self.econ), _native.ptr(self.evals), _native.ptr(y), self.npos,
            _native.ptr(out), _native.stream_handle(self.device)))
        return out

    def traces_dense(self, x, out):
        _native.check(self.lib.psd_sdls_traces_dense(
            _native.ptr(x), x.stride(0), _native.ptr(self.crow), _native.ptr(self.ccol),
            _native.ptr(self.cval), _native.ptr(self.cptr), self.m, _native.ptr(out),
            _native.stream_handle(self.device)))
        return out

    def traces(self, wd, w, r, out):
        _native.check(self.lib.psd_sdls_traces(
            _native.ptr(wd), _native.ptr(w), w.stride(0) if r else 1, r, _native.ptr(self.crow),
            _native.ptr(self.ccol), _native.ptr(self.cval), _native.ptr(self.cptr), self.m,
            _native.ptr(out), _native.stream_handle(self.device)))
        return out


def _scale_columns(lib, w, d, device):
    out = torch.empty_like(w)
    if w.shape[1]:
        _native.check(lib.psd_scale_columns(_native.ptr(w), w.stride(0), _native.ptr(d),
                                            _native.ptr(out), out.stride(0), w.shape[0],
                                            w.shape[1], _native.stream_handle(device)))
    return out


def _factored_projection(x_dual, n, cfg, rng, lib, plan, device, fw, fd, alpha):
    """One projection (projection.py:180-223 semantics inside solve): factors only."""
    params = cfg.params
    width = params.width
    if width > n:
        raise errors.error("InvalidParams", f"k+l = {width} exceeds min(m, n) = {n}")
    om = draw_gaussian(rng, (n, width), device)
    rep = _native.PsdReport()
    # the library's symmetry pass (x_dual is bitwise symmetric by construction) also
    # yields the INT8 engine's row scales, so it costs no extra read of X
    flags = 0
    _native.check(lib.psd_ran_proj(plan.handle, _native.ptr(x_dual), n, n, _native.ptr(om),
                                   om.stride(0), params.k, params.l, params.q, float(alpha), flags,
                                   ctypes.c_void_p(0), n, _native.ptr(fw), width, _native.ptr(fd),
                                   ctypes.byref(rep), _native.stream_handle(device)))
    return rep.effective_rank


def solve(problem, proj=None, *, beta=0.5, epsilon=1e-8, max_iter=100, y0=None, rng=None,
          alpha_refresh=1, keep_trajectory=False, exact_check_dim=2000, device=None):
    """sdls.py:164-265 on the GPU.  ``proj`` is this package's ``ProjectorConfig``
    or the reference's (after ``install()``); the default is the exact projector,
    as in the reference.  Randomized / scaled projectors keep X₊ factored inside
    the loop; exact / polar form it densely (full eigensolve on the device)."""
    if epsilon <= 0 or beta <= 0 or max_iter < 1:
        raise errors.error("InvalidParams", "need epsilon > 0, beta > 0, max_iter >= 1")
    proj = proj or ProjectorConfig(method="exact")
    rng = rng_from_seed(rng)
    if proj.method in ("exact", "polar"):
        return _solve_dense(problem, proj, beta, epsilon, max_iter, y0, rng, keep_trajectory,
                            device)
    t0 = time.perf_counter()
    prob = SparseSdlsProblem.from_reference(problem)
    dev = torch.device(device) if device else default_device()
    lib = _native.load_library()
    dp = _DeviceProblem(prob, dev)
    n, m = prob.n, prob.m
    scaled = proj.method == "scaled_randomized"
    width = proj.params.width
    plan = _native.get_plan(n, width, dev)
    x_dual = torch.empty((n, n), dtype=torch.float64, device=dev)
    fw = torch.empty((n, width), dtype=torch.float64, device=dev)
    fd = torch.empty(width, dtype=torch.float64, device=dev)
    t = torch.empty(m, dtype=torch.float64, device=dev)
    grad = torch.zeros(m, dtype=torch.float64, device=dev)
    nrm = torch.zeros(1, dtype=torch.float64, device=dev)
    if m == 0:  # sdls.py:198-210
        dp.assemble(torch.zeros(1, dtype=torch.float64, device=dev), x_dual)
        from .projection import project
        res = project(x_dual, proj, rng).result
        misfit = res - dp.cr
        return SolveReport(res.cpu().numpy(), np.zeros(0), 0, 0.0, 0.0,
                           0.5 * float((misfit * misfit).sum().item()), proj.method, True,
                           time.perf_counter() - t0)

    if y0 is None and isinstance(rng, DeviceRng):      # perf mode: device Philox stream
        y = rng.normal(m, dev).clone()
    else:
        y_host = rng.standard_normal(m) if y0 is None else np.asarray(y0, dtype=float).ravel()  # :212
        if y_host.size != m:
            raise errors.error("DimensionMismatch", f"y has length {y_host.size}, expected m = {m}")
        y = torch.from_numpy(y_host.copy()).to(dev)
    trajectory = [] if keep_trajectory else None
    y_trajectory = [] if keep_trajectory else None
    iterations, converged, r = 0, False, 0
    alpha_cached = None
    for it in range(1, max_iter + 1):                                # sdls.py:221-245
        dp.assemble(y, x_dual)
        alpha = 0.0
        if scaled:
            op = Operand(x_dual, "torch_cuda", dev)
            if proj.alpha_override is not None:
                alpha_cached = float(proj.alpha_override)
            elif alpha_cached is None or (it - 1) % max(1, alpha_refresh) == 0:
                alpha_cached = min_eig_magnitude_device(op, proj.power_N, rng)
            alpha = alpha_cached * proj.scale_factor
            mx = torch.zeros(1, dtype=torch.float64, device=dev)
            _native.check(lib.psd_max_abs(_native.ptr(x_dual), n, n, n, _native.ptr(mx),
                                          _native.stream_handle(dev)))
            if alpha <= ALPHA_TOL_FACTOR * max(1.0, mx.item()):       # AlphaTooSmall → unscaled
                alpha = 0.0
        if keep_trajectory:
            y_trajectory.append(y.cpu().numpy())
        r = _factored_projection(x_dual, n, proj, rng, lib, plan, dev, fw, fd, alpha)
        wd = _scale_columns(lib, fw[:, :r], fd[:r], dev) if r else fw[:, :0]
        dp.traces(wd.contiguous(), fw[:, :r].contiguous() if r else fw, r, t)
        _native.check(lib.psd_sdls_step(_native.ptr(dp.b), _native.ptr(t), _native.ptr(y),
                                        _native.ptr(grad), m, float(beta), float(epsilon),
                                        _native.ptr(nrm), _native.stream_handle(dev)))
        grad_norm = float(nrm.item())
        iterations = it
        if keep_trajectory:
            trajectory.append(TrajectoryPoint(it, grad_norm, grad_norm))
        if grad_norm <= epsilon:
            converged = True
            break

    w_last = fw[:, :r].contiguous()
    d_last = fd[:r].contiguous()
    x_current = reconstruct_device(w_last, d_last, n, dev)
    misfit = x_current - dp.cr
    objective = 0.5 * float((misfit * misfit).sum().item())
    objective -= float(torch.dot(y, t - dp.b).item())                # sdls.py:103-108
    exact_residual = None
    if n <= exact_check_dim:                                          # sdls.py:247-250
        dp.assemble(y, x_dual)
        _, vals, vecs, re = exact_psd_projection_device(Operand(x_dual, "torch_cuda", dev),
                                                        validate=False)
        te = torch.empty(m, dtype=torch.float64, device=dev)
        ve = vecs[:, :re].contiguous()
        dp.traces(_scale_columns(lib, ve, vals[:re].contiguous(), dev).contiguous(), ve, re, te)
        exact_residual = float(torch.linalg.vector_norm(te - dp.b).item())
    return SolveReport(
        x_solution=x_current.cpu().numpy(),
        y_final=y.cpu().numpy(),
        iterations=iterations,
        grad_norm_final=float(torch.linalg.vector_norm(grad).item()),
        feasibility_residual=float(torch.linalg.vector_norm(t - dp.b).item()),
        objective=objective,
        projection_method=proj.method,
        converged=converged,
        wall_time=time.perf_counter() - t0,
        trajectory=trajectory,
        y_trajectory=y_trajectory,
        exact_feasibility_residual=exact_residual,
    )


def _solve_dense(problem, proj, beta, epsilon, max_iter, y0, rng, keep_trajectory, device):
    """sdls.py:189-265 with the exact / polar projector: per iteration the dual
    matrix is assembled on the device, projected densely by ``project`` (device
    eigensolve, projection.py:162-177), and Tr(AᵢX₊) is read from the dense X₊ on
    the constraint nonzeros (``psd_sdls_traces_dense``).  No RNG is drawn except
    y₀ (sdls.py:212); the exact-residual check only applies to randomized runs
    (sdls.py:247)."""
    from .projection import project
    t0 = time.perf_counter()
    prob = SparseSdlsProblem.from_reference(problem)
    dev = torch.device(device) if device else default_device()
    lib = _native.load_library()
    dp = _DeviceProblem(prob, dev)
    n, m = prob.n, prob.m
    x_dual = torch.empty((n, n), dtype=torch.float64, device=dev)
    if m == 0:
        dp.assemble(torch.zeros(1, dtype=torch.float64, device=dev), x_dual)
        res = project(x_dual, proj, rng).result
        misfit = res - dp.cr
        return SolveReport(res.cpu().numpy(), np.zeros(0), 0, 0.0, 0.0,
                           0.5 * float((misfit * misfit).sum().item()), proj.method, True,
                           time.perf_counter() - t0)
    y_host = rng.standard_normal(m) if y0 is None else np.asarray(y0, dtype=float).ravel()
    if y_host.size != m:
        raise errors.error("DimensionMismatch", f"y has length {y_host.size}, expected m = {m}")
    y = torch.from_numpy(y_host.copy()).to(dev)
    t = torch.empty(m, dtype=torch.float64, device=dev)
    grad = torch.zeros(m, dtype=torch.float64, device=dev)
    nrm = torch.zeros(1, dtype=torch.float64, device=dev)
    trajectory = [] if keep_trajectory else None
    y_trajectory = [] if keep_trajectory else None
    iterations, converged, x_current = 0, False, None
    for it in range(1, max_iter + 1):                                # sdls.py:221-245
        dp.assemble(y, x_dual)
        if keep_trajectory:
            y_trajectory.append(y.cpu().numpy())
        x_current = project(x_dual, proj, rng).result
        dp.traces_dense(x_current, t)
        _native.check(lib.psd_sdls_step(_native.ptr(dp.b), _native.ptr(t), _native.ptr(y),
                                        _native.ptr(grad), m, float(beta), float(epsilon),
                                        _native.ptr(nrm), _native.stream_handle(dev)))
        grad_norm = float(nrm.item())
        iterations = it
        if keep_trajectory:
            trajectory.append(TrajectoryPoint(it, grad_norm, grad_norm))
        if grad_norm <= epsilon:
            converged = True
            break
    misfit = x_current - dp.cr
    objective = 0.5 * float((misfit * misfit).sum().item())
    objective -= float(torch.dot(y, t - dp.b).item())                # sdls.py:103-108
    return SolveReport(
        x_solution=x_current.cpu().numpy(),
        y_final=y.cpu().numpy(),
        iterations=iterations,
        grad_norm_final=float(torch.linalg.vector_norm(grad).item()),
        feasibility_residual=float(torch.linalg.vector_norm(t - dp.b).item()),
        objective=objective,
        projection_method=proj.method,
        converged=converged,
        wall_time=time.perf_counter() - t0,
        trajectory=trajectory,
        y_trajectory=y_trajectory,
    )
