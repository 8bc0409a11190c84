"""Randomized PSD projections on the GPU — drop-in for psdcone/projection.py.

``ran_proj`` (Alg. 2, projection.py:92-119), ``ran_proj_scal`` (Alg. 3,
projection.py:122-159) and the ``project`` dispatcher (projection.py:180-223)
keep the reference signatures, validation order, RNG draw order and report
fields.  All arithmetic runs in libpsdproj.so (FP64 DMMA tensor-core GEMMs,
CholeskyQR, block-Jacobi eigensolver, mirrored SYRK reconstruction); numpy
inputs are uploaded once and results copied back, torch CUDA inputs stay on
the device.  Extra keyword-only arguments: ``omega=`` (inject Ω),
``assume_symmetric=`` (skip the validation pass for inputs known to be
bitwise symmetric), ``dtype=`` ("fp64" default — the reference's float64
semantics; "fp32" — the FP32 path: 3xTF32 tcgen05 GEMMs, FP64 QR/eigh,
fp32 result, parity ≤1e-4 against the FP64 oracle on the fp32-rounded X).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import torch

from . import _native, errors
from ._tensors import as_device, draw_gaussian, require_square
from .sketch import RangeParams, min_eig_magnitude_device
from .symmetric import check_symmetric_device, eigh_device, reconstruct_device, rng_from_seed

METHODS = ("exact", "polar", "randomized", "scaled_randomized")  # projection.py:21
ALPHA_TOL_FACTOR = 1e-12  # projection.py:133


@dataclass
class ProjectorConfig:
    """projection.py:24-49."""

    method: str = "exact"
    params: RangeParams | None = None
    power_N: int = 10
    alpha_override: float | None = None
    scale_factor: float = 1.0
    collect_diagnostics: bool = False
    return_factors: bool = False
    dtype: str = "fp64"

    def __post_init__(self):
        self.dtype = resolve_dtype(self.dtype)
        if self.method not in METHODS:
            raise errors.error("InvalidParams", f"unknown projection method {self.method!r}")
        if self.method in ("randomized", "scaled_randomized") and self.params is None:
            raise errors.error("InvalidParams", f"method {self.method!r} requires RangeParams")
        if self.method == "scaled_randomized" and self.alpha_override is None and self.power_N < 1:
            raise errors.error("InvalidParams", "scaled method needs power_N >= 1 or alpha_override")


@dataclass
class ProjectionReport:
    """projection.py:52-69 (+ ``device_info``: kernel-side diagnostics)."""

    result: object
    method: str
    effective_rank: int
    alpha_used: float | None = None
    residual_frob: float | None = None
    wall_time: float = 0.0
    factors: tuple | None = None
    fallback: bool = False
    basis_width: int = 0
    device_info: dict | None = field(default=None, repr=False)


def resolve_dtype(dtype):
    """None / fp64 / float64 → "fp64"; fp32 / float32 → "fp32"."""
    if dtype is None:
        return "fp64"
    name = str(dtype).replace("torch.", "").replace("numpy.", "").lower()
    if name in ("fp64", "float64", "double", "f64", "<class 'numpy.float64'>"):
        return "fp64"
    if name in ("fp32", "float32", "float", "f32", "<class 'numpy.float32'>"):
        return "fp32"
    raise errors.error("InvalidParams", f"unsupported dtype {dtype!r} (fp64 or fp32)")


_FP64_ENGINE = "auto"
INT8_MIN_N = 3072   # "auto": INT8 emulation from this n up (measured crossover)


def set_fp64_engine(engine):
    """Tensor-core engine of the FP64 n×n products: "auto" (default: FP64 emulated
    exactly on the INT8 tensor cores, Ozaki scheme II, for n ≥ 3072; DMMA below),
    "int8" (emulation at any n) or "dmma" (the FP64 DMMA kernel).  Returns the
    previous setting."""
    global _FP64_ENGINE
    if engine not in ("auto", "int8", "dmma"):
        raise errors.error("InvalidParams", f"unknown FP64 engine {engine!r} (auto, int8 or dmma)")
    prev, _FP64_ENGINE = _FP64_ENGINE, engine
    return prev


def _operand(x, dtype):
    return as_device(x, dtype=torch.float32 if resolve_dtype(dtype) == "fp32" else torch.float64)


def _validate_in_library(op, assume_symmetric):
    """require_symmetric (symmetric.py:39-57, at projection.py:100/:132) and the
    alpha_tol test (projection.py:133-137) run inside psd_ran_proj[_f32] — its
    symmetry pass also yields the row scales of the INT8 engine, so X is read once
    for both.  ``assume_symmetric`` (FP64 only) skips the pass: the caller
    guarantees a bitwise-symmetric X."""
    return op.t.dtype == torch.float32 or not assume_symmetric


def _result_buffer(out, n, op):
    """``out=`` of ran_proj / ran_proj_scal: a contiguous n×n CUDA tensor of X's dtype."""
    if out is None:
        return torch.empty((n, n), dtype=op.t.dtype, device=op.device)
    if (not isinstance(out, torch.Tensor) or not out.is_cuda or out.device != op.device
            or out.dtype != op.t.dtype or tuple(out.shape) != (n, n) or not out.is_contiguous()):
        raise errors.error("InvalidParams", f"out must be a contiguous {n}x{n} {op.t.dtype} tensor on {op.device}")
    return out


def _prefetch_hint(lib, plan, prefetch, n, op):
    """psd_plan_prefetch: ``prefetch`` is the matrix the NEXT call will project (a pipelined
    batch — its validation and INT8 residue planes are prepared on a side stream while this
    call's CholeskyQR / eigensolver run).  FP64 n×n contiguous CUDA tensors only; anything
    else clears the hint."""
    ok = (isinstance(prefetch, torch.Tensor) and prefetch.is_cuda and prefetch.device == op.device
          and prefetch.dtype == op.t.dtype and tuple(prefetch.shape) == (n, n) and prefetch.stride(1) == 1)
    entry = lib.psd_plan_prefetch_f32 if op.t.dtype == torch.float32 else lib.psd_plan_prefetch
    _native.check(entry(plan.handle, _native.ptr(prefetch) if ok else None, n,
                        prefetch.stride(0) if ok else n))
    plan.prefetch_ref = prefetch if ok else None   # keep the tensor alive until it is consumed


def _run(op, n, params, om, alpha, validate, collect_diagnostics, return_factors, method, t0, out=None,
         prefetch=None):
    width = params.width
    lib = _native.load_library()
    plan = _native.get_plan(n, min(width, n), op.device)   # width > n: raised after the symmetry check
    if prefetch is not None or getattr(plan, "prefetch_ref", None) is not None:
        _prefetch_hint(lib, plan, prefetch, n, op)
    dev = op.device
    f32 = op.t.dtype == torch.float32
    result = _result_buffer(out, n, op)
    fw = torch.empty((n, width), dtype=torch.float64, device=dev) if return_factors else None
    fd = torch.empty(width, dtype=torch.float64, device=dev) if return_factors else None
    if f32:
        flags = 0  # psd_ran_proj_f32 runs require_symmetric / alpha_tol on the fp32 X
        om = om.to(torch.float32).contiguous()
    else:
        flags = 0 if validate else _native.FLAG_SKIP_SYMCHECK | _native.FLAG_ASSUME_SYMMETRIC
        if _FP64_ENGINE == "dmma":
            flags |= _native.FLAG_FP64_DMMA
        elif _FP64_ENGINE == "int8":
            flags |= _native.FLAG_FP64_INT8
    if collect_diagnostics:
        flags |= _native.FLAG_DIAGNOSTICS
    rep = _native.PsdReport()
    entry = lib.psd_ran_proj_f32 if f32 else lib.psd_ran_proj
    _native.check(entry(plan.handle, _native.ptr(op.t), n, n, _native.ptr(om),
                        om.stride(0), params.k, params.l, params.q, float(alpha), flags,
                        _native.ptr(result), n, _native.ptr(fw), width, _native.ptr(fd),
                        ctypes.byref(rep), _native.stream_handle(dev)))
    r = rep.effective_rank
    factors = None
    if return_factors:
        factors = (op.give_back(fw[:, :r].contiguous()), op.give_back(fd[:r].contiguous()))
    info = rep.as_dict()
    return ProjectionReport(
        result=op.give_back(result),
        method=method,
        effective_rank=int(r),
        alpha_used=float(alpha) if alpha > 0 else None,
        residual_frob=float(rep.residual_frob) if collect_diagnostics and not f32 else None,
        wall_time=time.perf_counter() - t0,
        factors=factors,
        basis_width=int(rep.basis_width),
        device_info=info,
    )


def _ran_proj_op(op, params, rng, collect_diagnostics, return_factors, omega, validate, t0, out=None,
                 prefetch=None):
    n = require_square(op)
    width = params.width
    if width > n and not validate:   # sketch.py:67-69 (else raised by the library after its check)
        raise errors.error("InvalidParams", f"k+l = {width} exceeds min(m, n) = {n}")
    om = as_device(omega, op.device).t if omega is not None else draw_gaussian(rng, (n, width), op.device)
    return _run(op, n, params, om, 0.0, validate, collect_diagnostics, return_factors, "randomized", t0,
                out, prefetch)


def ran_proj(x, params, rng, collect_diagnostics=False, return_factors=False, *, omega=None,
             assume_symmetric=False, dtype=None, out=None, prefetch=None):
    """projection.py:92-119 (Alg. 2): X̂₊ = Q U D₊ Uᵀ Qᵀ.

    ``prefetch`` (extension for batches of projections): the device matrix the next
    ``ran_proj`` call will project; see psd_plan_prefetch (include/psdproj.h)."""
    t0 = time.perf_counter()
    op = _operand(x, dtype)
    require_square(op)
    validate = _validate_in_library(op, assume_symmetric)      # projection.py:100
    return _ran_proj_op(op, params, rng, collect_diagnostics, return_factors, omega, validate, t0, out,
                        prefetch)


def _ran_proj_scal_op(op, params, alpha, rng, collect_diagnostics, return_factors, omega, validate, t0,
                      out=None):
    n = require_square(op)
    if not validate:  # assume_symmetric: the library skips its pass, alpha_tol needs max|x| here
        max_abs = check_symmetric_device(op).max_abs
        alpha_tol = ALPHA_TOL_FACTOR * max(1.0, max_abs)            # projection.py:133
        if alpha <= alpha_tol:
            raise errors.error(
                "AlphaTooSmall",
                f"alpha = {alpha:.3e} is at or below tolerance {alpha_tol:.3e}; input is numerically PSD")
    width = params.width
    if width > n and not validate:
        raise errors.error("InvalidParams", f"k+l = {width} exceeds min(m, n) = {n}")
    om = as_device(omega, op.device).t if omega is not None else draw_gaussian(rng, (n, width), op.device)
    return _run(op, n, params, om, float(alpha), validate, collect_diagnostics, return_factors,
                "scaled_randomized", t0, out)


def ran_proj_scal(x, params, alpha, rng, collect_diagnostics=False, return_factors=False, *,
                  omega=None, assume_symmetric=False, dtype=None, out=None):
    """projection.py:122-159 (Alg. 3) through B = (X + αI)/α (fused in the GEMM epilogues)."""
    t0 = time.perf_counter()
    op = _operand(x, dtype)
    require_square(op)
    validate = _validate_in_library(op, assume_symmetric)
    return _ran_proj_scal_op(op, params, alpha, rng, collect_diagnostics, return_factors, omega,
                             validate, t0, out)


def _exact_report(op, method, t0):
    """projection.py:162-177 on the GPU (eigh + mirrored reconstruction)."""
    n = op.t.shape[0]
    vals, vecs = eigh_device(op, validate=False)
    r = int((vals > 0.0).sum().item())
    if method == "exact":
        result = reconstruct_device(vecs[:, :r], vals[:r], n, op.device)
    else:
        # polar form (X + (XᵀX)^½)/2 = (X + V|Λ|Vᵀ)/2 for symmetric X (symmetric.py:117-128)
        absr = reconstruct_device(vecs, vals.abs(), n, op.device)
        result = (op.t + absr) / 2.0
        result = (result + result.T) / 2.0
    factors = None
    if method == "exact":
        factors = (op.give_back(vecs[:, :r].contiguous()), op.give_back(vals[:r].contiguous()))
    return ProjectionReport(result=op.give_back(result), method=method, effective_rank=r,
                            wall_time=time.perf_counter() - t0, factors=factors, basis_width=n)


def config_dtype(cfg):
    """Compute dtype of a config.  The reference's ``ProjectorConfig``
    (projection.py:24-49) has no ``dtype`` field: after ``install()`` its
    instances reach this dispatcher and run the reference's float64 semantics."""
    return resolve_dtype(getattr(cfg, "dtype", None))


def project(x, cfg, rng=None, *, omega=None, assume_symmetric=False):
    """projection.py:180-223: dispatcher with the scaled → unscaled AlphaTooSmall fallback.
    ``cfg`` is this package's ``ProjectorConfig`` or the reference's own."""
    t0 = time.perf_counter()
    op = _operand(x, config_dtype(cfg))
    require_square(op)
    # require_symmetric (projection.py:189): the dense methods validate here; the
    # randomized ones inside the library call (with the same exceptions)
    validate = _validate_in_library(op, assume_symmetric)
    if cfg.method in ("exact", "polar"):
        if op.t.dtype != torch.float32 and validate:
            check_symmetric_device(op)
        if op.t.dtype == torch.float32:  # dense eigh stays FP64; result handed back as fp32
            op64 = type(op)(op.t.double(), op.kind, op.device)
            check_symmetric_device(op64)
            rep = _exact_report(op64, cfg.method, t0)
            rep.result = op.give_back(torch.as_tensor(rep.result, device=op.device).to(torch.float32))
            return rep
        return _exact_report(op, cfg.method, t0)

    rng = rng_from_seed(rng if rng is not None else (cfg.params.seed if cfg.params else None))
    if cfg.method == "randomized":
        report = _ran_proj_op(op, cfg.params, rng, cfg.collect_diagnostics, cfg.return_factors,
                              omega, validate, t0)
        report.wall_time = time.perf_counter() - t0
        return report

    if cfg.alpha_override is not None:
        alpha = float(cfg.alpha_override)
    elif op.t.dtype == torch.float32:  # α estimate on the fp32 values, in FP64
        alpha = min_eig_magnitude_device(type(op)(op.t.double(), op.kind, op.device), cfg.power_N, rng)
    else:
        # require_symmetric first, as the reference does (projection.py:189); a bitwise-symmetric
        # X lets the 2(N+1) products of the estimate read only its lower triangle
        bitwise = check_symmetric_device(op).bitwise if validate else True
        alpha = min_eig_magnitude_device(op, cfg.power_N, rng, bitwise_symmetric=bitwise)   # :206
    alpha *= cfg.scale_factor
    try:
        report = _ran_proj_scal_op(op, cfg.params, alpha, rng, cfg.collect_diagnostics,
                                   cfg.return_factors, omega, validate, t0)
    except errors.REGISTRY["AlphaTooSmall"]:
        report = _ran_proj_op(op, cfg.params, rng, cfg.collect_diagnostics, cfg.return_factors,
                              omega, validate, t0)
        report.fallback = True
        report.alpha_used = float(alpha)
    report.wall_time = time.perf_counter() - t0
    return report


def flops(n, params, effective_rank):
    """Algorithmic FLOPs of one projection: 2n²w(2q+2) + n²r₊."""
    return 2.0 * n * n * params.width * (2 * params.q + 2) + float(n) * n * effective_rank


__all__ = ["METHODS", "resolve_dtype", "ProjectorConfig", "ProjectionReport", "ran_proj", "ran_proj_scal",
           "project", "flops", "set_fp64_engine"]
