"""CPU oracle for the randomized PSD-cone projection hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may call it, and there only as
the checker (or the timed CPU baseline), never as the thing measured or
shipped.

This is a numpy restatement of the reference ``psdcone`` package
(``/root/reference/pkg/src/psdcone``, pure Python over numpy/OpenBLAS/LAPACK,
numpy unpinned ``>=1.24`` per ``pkg/pyproject.toml:10``).  It performs the
same numpy calls in the same order as the reference, so on identical inputs it
reproduces the reference bit-for-bit in the same container.  The only change
is that every random draw can be *injected* (``omega=`` / ``v0=``) so that the
GPU path and the oracle consume identical Gaussian test matrices; when a
``numpy.random.Generator`` is passed instead, draws happen in the reference's
order (``Ω`` after the two power-iteration start vectors).

Parity pin: ``tests/golden/make_golden.py`` imports the real reference in
this container and writes fixtures (inputs, Ω, outputs) to
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against every fixture (bit-exact / ≤1e-13 relative).  The GPU box has no
``/root/reference``; it uses only the committed fixtures.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SYM_TOL_FACTOR = 1e-10          # symmetric.py:16
RANK_TRUNCATION_FACTOR = 1e-12  # sketch.py:12
ALPHA_TOL_FACTOR = 1e-12        # projection.py:133


class OracleError(Exception):
    """Raised where the reference raises a PsdconeError subclass; ``kind`` names it."""

    def __init__(self, kind, msg=""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------- symcore ---

def symmetrize(a):
    """(A + Aᵀ)/2 — symmetric.py:31-36."""
    a = np.asarray(a, dtype=float)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise OracleError("NonSquareError", str(a.shape))
    return (a + a.T) / 2.0


def require_symmetric(a, tol=None):
    """symmetric.py:39-57: tol = 1e-10·max(1, max|a|); defect = max|a − aᵀ|."""
    a = np.asarray(a, dtype=float)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise OracleError("NonSquareError", str(a.shape))
    if a.shape[0] < 1:
        raise OracleError("NonSquareError", "dimension must be >= 1")
    if tol is None:
        tol = SYM_TOL_FACTOR * max(1.0, float(np.max(np.abs(a))) if a.size else 1.0)
    defect = float(np.max(np.abs(a - a.T))) if a.size else 0.0
    if defect > tol:
        raise OracleError("AsymmetricMatrixError", f"{defect:.3e} > {tol:.3e}")
    return a


def symmetry_stats(a):
    """(max|a|, max|a−aᵀ|) — the two reductions of symmetric.py:51-52."""
    a = np.asarray(a, dtype=float)
    return float(np.max(np.abs(a))), float(np.max(np.abs(a - a.T)))


@dataclass(frozen=True)
class EigenDecomposition:
    values: np.ndarray
    vectors: np.ndarray


def eigh(x):
    """symmetric.py:68-86: LAPACK syevd, descending, largest-|entry| positive."""
    x = require_symmetric(x)
    try:
        w, v = np.linalg.eigh(x)
    except np.linalg.LinAlgError as exc:  # pragma: no cover - LAPACK failure
        raise OracleError("ConvergenceFailure", str(exc)) from exc
    w = w[::-1].copy()
    v = v[:, ::-1].copy()
    anchor = np.argmax(np.abs(v), axis=0)
    signs = np.sign(v[anchor, np.arange(v.shape[1])])
    signs[signs == 0] = 1.0
    v *= signs
    return EigenDecomposition(values=w, vectors=v)


def exact_psd_projection(x):
    """symmetric.py:109-114 (used only as a test oracle)."""
    dec = eigh(x)
    clipped = np.maximum(dec.values, 0.0)
    proj = (dec.vectors * clipped) @ dec.vectors.T
    return (proj + proj.T) / 2.0


def polar_psd_projection(x):
    """symmetric.py:117-128: (X + (XᵀX)^½)/2 with the root from eigh(sym(XᵀX))."""
    x = require_symmetric(x)
    dec = eigh(symmetrize(x.T @ x))
    root = (dec.vectors * np.sqrt(np.maximum(dec.values, 0.0))) @ dec.vectors.T
    return symmetrize((x + root) / 2.0)


def rng_from_seed(seed):
    """symmetric.py:19-28."""
    if isinstance(seed, np.random.Generator):
        return seed
    return np.random.default_rng(seed)


def gaussian_matrix(rows, cols, rng):
    """symmetric.py:131-135."""
    return rng.standard_normal((rows, cols))


# ----------------------------------------------------------------- sketch ---

def range_finder(x, k, l, q, rng=None, omega=None, strict=False):
    """sketch.py:53-93 (Alg. 1 + power scheme + truncated economy QR).

    ``omega`` (n×(k+l)) replaces the draw at sketch.py:75 when given.
    Returns (basis, keep_mask, r_diag, frob_norm_of_Y).
    """
    x = np.asarray(x, dtype=float)
    m, n = x.shape
    width = k + l
    if width > min(m, n):
        raise OracleError("InvalidParams", f"k+l={width} > {min(m, n)}")
    stabilize = q >= 2                                          # sketch.py:74
    if omega is None:
        omega = gaussian_matrix(n, width, rng)
    y = x @ omega                                               # sketch.py:75
    for _ in range(q):                                          # sketch.py:76-82
        if stabilize:
            y = np.linalg.qr(y, mode="reduced")[0]
        z = x.T @ y
        if stabilize:
            z = np.linalg.qr(z, mode="reduced")[0]
        y = x @ z
    scale = np.linalg.norm(y)                                   # sketch.py:84
    q_full, r_full = np.linalg.qr(y, mode="reduced")            # sketch.py:85
    rdiag = np.abs(np.diag(r_full))
    keep = rdiag > RANK_TRUNCATION_FACTOR * scale               # sketch.py:86
    if not np.all(keep):
        if strict:
            raise OracleError("RankDeficientSample", f"rank {int(np.count_nonzero(keep))} < {width}")
        q_full = q_full[:, keep]
    return q_full, keep, rdiag, float(scale)


def power_iteration(x, n_iter, rng=None, v0=None):
    """sketch.py:96-114 (Alg. 4).  ``v0`` replaces the draw at :106."""
    x = np.asarray(x, dtype=float)
    if n_iter < 1:
        raise OracleError("InvalidParams", "n_iter >= 1")
    v = rng.standard_normal(x.shape[0]) if v0 is None else np.asarray(v0, dtype=float)
    floor = np.finfo(float).tiny * x.shape[0]
    for _ in range(n_iter):
        w = x @ v
        nrm = np.linalg.norm(w)
        if nrm <= floor:
            return 0.0
        v = w / nrm
    return float(np.linalg.norm(x @ v))


def min_eig_magnitude(x, n_iter, rng=None, v1=None, v2=None):
    """sketch.py:117-129 (Alg. 5): |σ₁ − PI(X − σ₁I)|, shifted matrix materialised."""
    x = np.asarray(x, dtype=float)
    s1 = power_iteration(x, n_iter, rng, v0=v1)
    shifted = x - s1 * np.eye(x.shape[0])
    s2 = power_iteration(shifted, n_iter, rng, v0=v2)
    return abs(s1 - s2)


# ------------------------------------------------------------- projection ---

@dataclass
class OracleReport:
    result: np.ndarray
    effective_rank: int
    basis_width: int
    alpha_used: float | None = None
    fallback: bool = False
    residual_frob: float | None = None
    factors: tuple | None = None
    basis: np.ndarray | None = None
    eigenvalues: np.ndarray | None = None


def _assemble_clipped(basis, vectors, clipped, scale=1.0):
    """projection.py:72-78."""
    w = basis @ vectors
    keep = clipped > 0.0
    w_kept = w[:, keep]
    d_kept = clipped[keep] * scale
    return symmetrize((w_kept * d_kept) @ w_kept.T), w_kept, d_kept


def _zero(n):
    """projection.py:81-89."""
    return OracleReport(result=np.zeros((n, n)), effective_rank=0, basis_width=0,
                        factors=(np.zeros((n, 0)), np.zeros(0)))


def ran_proj(x, k, l, q, rng=None, omega=None, collect_diagnostics=False):
    """projection.py:92-119 (Alg. 2)."""
    x = require_symmetric(x)                                    # :100
    basis, _, _, _ = range_finder(x, k, l, q, rng, omega)       # :101
    if basis.shape[1] == 0:
        return _zero(x.shape[0])
    compressed = symmetrize(basis.T @ x @ basis)                # :104
    dec = eigh(compressed)                                      # :105
    clipped = np.maximum(dec.values, 0.0)                       # :106
    result, w, d = _assemble_clipped(basis, dec.vectors, clipped)
    residual = None
    if collect_diagnostics:
        residual = float(np.linalg.norm(x - basis @ (basis.T @ x)))  # :110
    return OracleReport(result=result, effective_rank=int(d.size), basis_width=basis.shape[1],
                        residual_frob=residual, factors=(w, d), basis=basis,
                        eigenvalues=dec.values)


def ran_proj_scal(x, k, l, q, alpha, rng=None, omega=None, collect_diagnostics=False):
    """projection.py:122-159 (Alg. 3)."""
    x = require_symmetric(x)
    alpha_tol = ALPHA_TOL_FACTOR * max(1.0, float(np.max(np.abs(x))))   # :133
    if alpha <= alpha_tol:
        raise OracleError("AlphaTooSmall", f"{alpha:.3e} <= {alpha_tol:.3e}")
    n = x.shape[0]
    b = (x + alpha * np.eye(n)) / alpha                         # :139
    basis, _, _, _ = range_finder(b, k, l, q, rng, omega)       # :140
    if basis.shape[1] == 0:
        return _zero(n)
    compressed = symmetrize(basis.T @ b @ basis)                # :143
    dec = eigh(compressed)
    clipped = np.maximum(dec.values - 1.0, 0.0)                 # :145
    result, w, d = _assemble_clipped(basis, dec.vectors, clipped, scale=alpha)
    residual = None
    if collect_diagnostics:
        residual = float(np.linalg.norm(x - basis @ (basis.T @ x)))
    return OracleReport(result=result, effective_rank=int(d.size), basis_width=basis.shape[1],
                        alpha_used=float(alpha), residual_frob=residual, factors=(w, d),
                        basis=basis, eigenvalues=dec.values)


def project_scaled(x, k, l, q, power_n=10, alpha_override=None, scale_factor=1.0,
                   rng=None, v1=None, v2=None, omega=None):
    """projection.py:180-223, scaled branch: α estimate, ×scale_factor, AlphaTooSmall fallback."""
    x = require_symmetric(x)
    if alpha_override is not None:
        alpha = float(alpha_override)
    else:
        alpha = min_eig_magnitude(x, power_n, rng, v1=v1, v2=v2)
    alpha *= scale_factor
    try:
        return ran_proj_scal(x, k, l, q, alpha, rng, omega)
    except OracleError as exc:
        if exc.kind != "AlphaTooSmall":
            raise
        rep = ran_proj(x, k, l, q, rng, omega)
        rep.fallback = True
        rep.alpha_used = float(alpha)
        return rep


# --------------------------------------------------------------- helpers ---

def rel_frob(a, b):
    """‖a − b‖_F / max(‖b‖_F, tiny) — the parity metric of BASELINE.json north_star."""
    nb = float(np.linalg.norm(b))
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b))) / max(nb, 1e-300)


def flops_per_projection(n, w, q, r_plus):
    """F = 2n²w(2q+2) + n²·r₊."""
    return 2.0 * n * n * w * (2 * q + 2) + float(n) * n * r_plus


def c1_matrix(seed=0, n=1000):
    """BASELINE config 1: Haar V, λ₁..₃₀ geomspace(1e2,1e-2), rest U[−1,0]; X = VΛVᵀ symmetrised."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    v = np.linalg.qr(g)[0]
    lam = np.concatenate([np.geomspace(1e2, 1e-2, 30), rng.uniform(-1.0, 0.0, n - 30)])
    x = (v * lam) @ v.T
    return (x + x.T) / 2.0


def wigner(n, seed=0):
    """BASELINE config 2: (G + Gᵀ)/(2√n), bitwise symmetric."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    return (g + g.T) / (2.0 * math.sqrt(n))


def c3_matrix(n, seed=0, rank=200):
    """BASELINE config 3 (host restatement used at reduced n by tests)."""
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((n, rank)))[0]
    w = np.linalg.qr(rng.standard_normal((n, rank)))[0]
    s = np.geomspace(1e3, 1.0, rank)
    t = rng.uniform(0.0, 10.0, rank)
    g = rng.standard_normal((n, n))
    e = (g + g.T) / (2.0 * math.sqrt(n))
    x = (u * s) @ u.T - (w * t) @ w.T + 1e-3 * e
    return (x + x.T) / 2.0
