"""CPU oracle for the solver loop that drives the projection (BASELINE config 5).

TEST INFRASTRUCTURE ONLY (see oracle/psd_oracle.py).  A numpy restatement of
``psdcone.sdls`` (/root/reference/pkg/src/psdcone/sdls.py) — dense constraint
stacks as in the reference and, for config 5 (m=20000 constraints, whose dense
stack would be 2.68 TB), a sparse-COO problem exposing the same
``assemble``/``traces`` contract, which is the rebinding BASELINE.md §2
prescribes for the CPU baseline.  Pinned by tests/golden/sdls_*.npz, produced by
running the real reference ``solve`` on small dense instances.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import psd_oracle as orc


class DenseProblem:
    """SdlsProblem (sdls.py:21-57): dense (m, n, n) stack."""

    def __init__(self, c, rho, a_stack, b):
        self.c = np.asarray(c, dtype=float)
        self.rho = float(rho)
        self.a_stack = np.asarray(a_stack, dtype=float)
        self.b = np.asarray(b, dtype=float)
        self.n = self.c.shape[0]
        self.m = self.b.size

    def assemble(self, y):
        """assemble_dual_matrix, sdls.py:83-89."""
        x = self.c / self.rho
        if self.m:
            x = x + np.einsum("m,mij->ij", y, self.a_stack)
        return x

    def traces(self, x):
        """constraint_traces, sdls.py:76-80."""
        if self.m == 0:
            return np.zeros(0)
        return np.einsum("mij,ij->m", self.a_stack, x)


class SparseProblem:
    """Same contract with constraints as COO triplets (every stored entry
    explicit, i.e. both (i,j) and (j,i) for off-diagonal pairs)."""

    def __init__(self, c, rho, con, rows, cols, vals, b):
        self.c = np.asarray(c, dtype=float)
        self.rho = float(rho)
        self.con = np.asarray(con, dtype=np.int64)
        self.rows = np.asarray(rows, dtype=np.int64)
        self.cols = np.asarray(cols, dtype=np.int64)
        self.vals = np.asarray(vals, dtype=float)
        self.b = np.asarray(b, dtype=float)
        self.n = self.c.shape[0]
        self.m = self.b.size

    def assemble(self, y):
        x = self.c / self.rho
        extra = np.zeros_like(x)
        np.add.at(extra, (self.rows, self.cols), y[self.con] * self.vals)
        return x + extra

    def traces(self, x):
        t = np.zeros(self.m)
        np.add.at(t, self.con, self.vals * x[self.rows, self.cols])
        return t


@dataclass
class OracleSolveReport:
    x_solution: np.ndarray
    y_final: np.ndarray
    iterations: int
    grad_norm_final: float
    feasibility_residual: float
    objective: float
    converged: bool
    trajectory: list
    y_trajectory: list
    exact_feasibility_residual: float | None = None


def _lagrangian(problem, x, y):
    """sdls.py:103-108."""
    misfit = x - problem.c / problem.rho
    value = 0.5 * float(np.sum(misfit * misfit))
    if problem.m:
        value -= float(y @ (problem.traces(x) - problem.b))
    return value


def solve(problem, method, k, l, q, *, power_n=10, scale_factor=1.0, beta=0.5, epsilon=1e-8,
          max_iter=100, y0=None, rng=None, alpha_refresh=1, exact_check_dim=2000):
    """sdls.py:164-265 (Alg. 6) with any projector: randomized / scaled, or the
    dense exact (projection.py:162-177, symmetric.py:109-114) / polar
    (symmetric.py:117-128) ones, which draw nothing but y₀."""
    rng = orc.rng_from_seed(rng)
    scaled = method == "scaled_randomized"
    y = rng.standard_normal(problem.m) if y0 is None else np.asarray(y0, dtype=float).copy()  # :212
    traj, ytraj = [], []
    x_current = None
    grad = np.zeros(problem.m)
    iterations = 0
    converged = False
    alpha_cached = None
    for it in range(1, max_iter + 1):                                   # :221-245
        x_dual = problem.assemble(y)
        if scaled:
            if alpha_cached is None or (it - 1) % max(1, alpha_refresh) == 0:
                alpha_cached = orc.min_eig_magnitude(x_dual, power_n, rng)
            rep = orc.project_scaled(x_dual, k, l, q, alpha_override=alpha_cached,
                                     scale_factor=scale_factor, rng=rng)
        elif method == "exact":
            rep = None
            x_current = orc.exact_psd_projection(x_dual)
        elif method == "polar":
            rep = None
            x_current = orc.polar_psd_projection(x_dual)
        else:
            rep = orc.ran_proj(x_dual, k, l, q, rng=rng)
        if rep is not None:
            x_current = rep.result
        grad = problem.b - problem.traces(x_current)
        grad_norm = float(np.linalg.norm(grad))
        iterations = it
        traj.append(grad_norm)
        ytraj.append(y.copy())
        if grad_norm <= epsilon:
            converged = True
            break
        y = y + beta * grad
    exact_residual = None
    if method not in ("exact", "polar") and problem.n <= exact_check_dim:    # :247-250
        x_exact = orc.exact_psd_projection(problem.assemble(y))
        exact_residual = float(np.linalg.norm(problem.traces(x_exact) - problem.b))
    return OracleSolveReport(
        x_solution=x_current, y_final=y, iterations=iterations,
        grad_norm_final=float(np.linalg.norm(grad)),
        feasibility_residual=float(np.linalg.norm(problem.traces(x_current) - problem.b)),
        objective=_lagrangian(problem, x_current, y), converged=converged,
        trajectory=traj, y_trajectory=ytraj, exact_feasibility_residual=exact_residual)


def config5_instance(n, m, nnz_per=4, seed=0, rank=10):
    """BASELINE config 5: A_i with `nnz_per` seeded off-diagonal
    N(0,1) entries mirrored; b = A(Z Zᵀ); C = Wigner + 2I; ρ = 1.  Returns a
    SparseProblem (SDLS C enters directly, C/ρ)."""
    rng = np.random.default_rng(seed)
    i = rng.integers(0, n, size=(m, nnz_per))
    j = rng.integers(0, n - 1, size=(m, nnz_per))
    j = np.where(j >= i, j + 1, j)                      # off-diagonal
    v = rng.standard_normal((m, nnz_per))
    con = np.repeat(np.arange(m), 2 * nnz_per)
    rows = np.stack([i, j], -1).reshape(m, -1)
    cols = np.stack([j, i], -1).reshape(m, -1)
    vals = np.repeat(v, 2, axis=1)
    z = rng.standard_normal((n, rank))
    x0 = z @ z.T
    g = rng.standard_normal((n, n))
    c = (g + g.T) / (2.0 * math.sqrt(n)) + 2.0 * np.eye(n)
    prob = SparseProblem(c, 1.0, con, rows.ravel(), cols.ravel(), vals.ravel(), np.zeros(m))
    prob.b = prob.traces(x0)
    return prob


def lipschitz_beta(problem, iters=50, seed=0):
    """β = 1/L with L = λ_max(⟨A_i, A_j⟩_F) by power iteration on the sparse Gram
    (SURVEY A8): the Gram action is v ↦ traces(assemble-of-v without C)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(problem.m)
    v /= np.linalg.norm(v)
    lam = 0.0
    c_saved = problem.c
    problem.c = np.zeros_like(c_saved)
    try:
        for _ in range(iters):
            w = problem.traces(problem.assemble(v))
            lam = float(np.linalg.norm(w))
            v = w / lam
    finally:
        problem.c = c_saved
    return 1.0 / lam
