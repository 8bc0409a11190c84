"""Monte-Carlo projection-error harness on the GPU — drop-in for
``psdcone.experiments.projection_error_sweep`` (experiments.py:78-137) and the
closed-form bounds it reports (bounds.py:19-221).

The benchmark matrix is generated on the host exactly as the reference does
(same numpy stream, experiments.py:34-42 → symmetric.py:138-153), uploaded
once; the exact projection (dense eigensolve), every randomized projection,
the Frobenius errors and the spectral errors (dense eigensolve of the
difference, symmetric.py:94-97) run on the GPU.  Ω is drawn from the
reference's numpy stream in the reference's order, so each trial projects
with the same Ω as the reference.  The bounds are scalar formulas of the
spectrum and stay on the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import errors
from ._tensors import Operand, as_device
from .projection import ran_proj, ran_proj_scal
from .sketch import RangeParams
from .symmetric import eigh_device, exact_psd_projection_device, rng_from_seed

FOUR_BLOCK_BETAS = (3.0, 1.0, 6.0, 2.0)   # experiments.py:31


# ----------------------------------------------------------------- matrices --

def four_block_eigenvalues(n, beta):
    """bounds.py:206-221: n/4 copies each of β3, β4, −β2, −β1 (descending)."""
    b1, b2, b3, b4 = (float(b) for b in beta)
    if not (b3 > b1 > b4 > b2 > 0):
        raise errors.error("InvalidParams", "betas must satisfy beta3 > beta1 > beta4 > beta2 > 0")
    if n % 4 != 0 or n < 4:
        raise errors.error("InvalidParams", f"n must be a positive multiple of 4, got {n}")
    return np.repeat([b3, b4, -b2, -b1], n // 4).astype(float)


def random_orthogonal(n, rng):
    """symmetric.py:138-144: Haar orthogonal matrix, QR of a Gaussian, sign-fixed."""
    g = rng.standard_normal((n, n))
    q, r = np.linalg.qr(g)
    signs = np.sign(np.diag(r))
    signs[signs == 0] = 1.0
    return q * signs


def spectrum_matrix(eigenvalues, rng):
    """symmetric.py:147-153: V diag(λ) Vᵀ for a random orthogonal V, symmetrised."""
    ev = np.asarray(eigenvalues, dtype=float).ravel()
    if ev.size < 1:
        raise ValueError("need at least one eigenvalue")
    y = random_orthogonal(ev.size, rng)
    m = (y * ev) @ y.T
    return (m + m.T) / 2.0


def four_block_matrix(n, beta=FOUR_BLOCK_BETAS, rng=None):
    """experiments.py:34-42 (host generation: the same matrix as the reference)."""
    return spectrum_matrix(four_block_eigenvalues(n, beta), rng_from_seed(rng))


# ------------------------------------------------------------------- bounds --

@dataclass(frozen=True)
class SpectrumSummary:
    """bounds.py:19-63 (descending eigenvalues / singular values)."""

    n: int
    eigenvalues: np.ndarray | None = None
    singular_values: np.ndarray | None = None

    @classmethod
    def from_eigenvalues(cls, eigenvalues):
        ev = np.sort(np.asarray(eigenvalues, dtype=float).ravel())[::-1]
        return cls(n=ev.size, eigenvalues=ev, singular_values=np.sort(np.abs(ev))[::-1])

    @property
    def sigmas(self):
        if self.singular_values is not None:
            return self.singular_values
        return np.sort(np.abs(self.eigenvalues))[::-1]


@dataclass(frozen=True)
class BoundParams:
    """bounds.py:66-87."""

    k: int
    l: int
    q: int = 0
    alpha: float | None = None

    def __post_init__(self):
        if self.k < 1:
            raise errors.error("InvalidParams", f"bounds require k >= 1, got {self.k}")
        if self.l < 2:
            raise errors.error("InvalidParams", f"bounds require l >= 2, got {self.l}")
        if self.q < 0:
            raise errors.error("InvalidParams", f"power exponent q must be >= 0, got {self.q}")


def _check_k(k, n):
    if not 1 <= k < n:
        raise errors.error("InvalidParams", f"need 1 <= k < n, got k = {k}, n = {n}")


def eps1(sigmas, k, l):
    """bounds.py:95-103: sqrt((1 + k/(l−1)) Σ_{j>k} σ_j²)."""
    s = np.asarray(sigmas, dtype=float).ravel()
    _check_k(k, s.size)
    return math.sqrt((1.0 + k / (l - 1.0)) * float(np.sum(s[k:] ** 2)))


def eps2(sigma_k_plus_1, k, l, q, n):
    """bounds.py:106-114."""
    _check_k(k, n)
    base = 1.0 + math.sqrt(k / (l - 1.0)) + math.e * math.sqrt(k + l) / l * math.sqrt(n - k)
    return base ** (1.0 / (2 * q + 1)) * float(sigma_k_plus_1)


def frob_bound_unscaled(spectrum, params):
    """bounds.py:117-122 (q = 0 only)."""
    if params.q != 0:
        raise errors.error("InvalidParams", "the Frobenius projection bound is only stated for q = 0")
    _check_k(params.k, spectrum.n)
    return (1.0 + math.sqrt(params.k + params.l)) * eps1(spectrum.sigmas, params.k, params.l)


def spectral_bound_unscaled(spectrum, params):
    """bounds.py:125-138."""
    sig = spectrum.sigmas
    _check_k(params.k, spectrum.n)
    s1 = float(sig[0])
    e2 = eps2(sig[params.k], params.k, params.l, params.q, spectrum.n)
    first = (1.0 + math.sqrt(spectrum.n)) * e2
    second = (1.0 + 4.0 / math.pi + (2.0 / math.pi) * math.log(2.0 * s1)) * e2 + \
        (1.0 / math.pi) * min(math.exp(-1.0), math.sqrt(2.0 * e2))
    return min(first, second)


def frob_bound_scaled(spectrum, params, alpha):
    """bounds.py:141-157 (q = 0 only)."""
    if params.q != 0:
        raise errors.error("InvalidParams", "the scaled Frobenius bound is only stated for q = 0")
    _check_k(params.k, spectrum.n)
    shifted = np.sort(spectrum.eigenvalues + alpha)[::-1]
    return alpha * math.sqrt(spectrum.n - params.k) + \
        (1.0 + math.sqrt(params.k + params.l)) * eps1(shifted, params.k, params.l)


def spectral_bound_scaled(spectrum, params, alpha):
    """bounds.py:160-178."""
    _check_k(params.k, spectrum.n)
    s1 = float(spectrum.sigmas[0])
    n = spectrum.n
    e2 = eps2(float(spectrum.eigenvalues[params.k]) + alpha, params.k, params.l, params.q, n)
    first = (1.0 + math.sqrt(n)) * (e2 + alpha / 2.0)
    second = (0.5 + 2.0 / math.pi + (1.0 / math.pi) * math.log(2.0 * s1)) * (2.0 * e2 + alpha) + \
        (1.0 / math.pi) * min(math.exp(-1.0), math.sqrt(2.0 * e2 + alpha))
    return min(first, second)


# -------------------------------------------------------------------- sweep --

@dataclass
class SweepRow:
    """experiments.py:66-75."""

    k: int
    method: str
    mean_frob_error: float
    mean_spectral_error: float
    frob_bound: float | None
    spectral_bound: float | None


def spectral_norm_device(d):
    """symmetric.py:94-97 on the GPU: max |λ| of the dense eigensolve."""
    vals, _ = eigh_device(Operand(d, "torch_cuda", d.device), validate=False)
    return float(vals.abs().max().item()) if vals.numel() else 0.0


def projection_error_sweep(n, beta, l, q, k_grid, trials, seed, alpha=None, compute_spectral=True,
                           *, device=None):
    """experiments.py:78-137 with every projection and error on the GPU."""
    beta = tuple(float(b) for b in beta)
    x_host = four_block_matrix(n, beta, rng_from_seed(seed))
    op = as_device(x_host, device)
    x = op.t
    x_plus = exact_psd_projection_device(op)[0]
    alpha = beta[0] if alpha is None else float(alpha)
    spectrum = SpectrumSummary.from_eigenvalues(four_block_eigenvalues(n, beta))
    rows = []
    for k in k_grid:
        params = RangeParams(k=int(k), l=int(l), q=int(q))
        errs = {"randomized": [], "scaled_randomized": []}
        for trial in range(trials):
            rng = rng_from_seed(seed + 1 + trial)
            plain = ran_proj(x, params, rng, assume_symmetric=True).result
            scal = ran_proj_scal(x, params, alpha, rng, assume_symmetric=True).result
            for tag, approx in (("randomized", plain), ("scaled_randomized", scal)):
                d = x_plus - approx
                frob = float(torch.linalg.vector_norm(d).item())
                spec = spectral_norm_device((d + d.T) / 2.0) if compute_spectral else float("nan")
                errs[tag].append((frob, spec))
        bp = BoundParams(k=int(k), l=int(l), q=int(q))
        frob_b = {"randomized": None, "scaled_randomized": None}
        if q == 0:
            frob_b["randomized"] = frob_bound_unscaled(spectrum, bp)
            frob_b["scaled_randomized"] = frob_bound_scaled(spectrum, bp, alpha)
        spec_b = {"randomized": spectral_bound_unscaled(spectrum, bp),
                  "scaled_randomized": spectral_bound_scaled(spectrum, bp, alpha)}
        for tag in ("randomized", "scaled_randomized"):
            arr = np.asarray(errs[tag])
            rows.append(SweepRow(k=int(k), method=tag, mean_frob_error=float(arr[:, 0].mean()),
                                 mean_spectral_error=float(arr[:, 1].mean()),
                                 frob_bound=frob_b[tag], spectral_bound=spec_b[tag]))
    return rows


__all__ = ["FOUR_BLOCK_BETAS", "four_block_eigenvalues", "random_orthogonal", "spectrum_matrix",
           "four_block_matrix", "SpectrumSummary", "BoundParams", "eps1", "eps2",
           "frob_bound_unscaled", "spectral_bound_unscaled", "frob_bound_scaled",
           "spectral_bound_scaled", "SweepRow", "spectral_norm_device", "projection_error_sweep"]
