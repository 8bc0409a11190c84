"""Generate golden fixtures by running the REAL reference ``psdcone`` package.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

Every fixture stores the inputs (X or the seed that regenerates it), the exact
random draws the reference consumed (Ω, power-iteration start vectors), and
the reference outputs.  The GPU box never reads ``/root/reference``; the
``-m gpu`` parity tests and ``smoke()`` use these committed ``.npz`` files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import psdcone  # noqa: E402  (the reference, imported read-only)
from psdcone import RangeParams, ProjectorConfig  # noqa: E402

from oracle import psd_oracle as orc  # noqa: E402


def _save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    clean = {}
    for k, v in arrays.items():
        if v is None:
            continue
        clean[k] = np.asarray(v)
    np.savez_compressed(path, **clean)
    print(f"wrote {name}: {sorted(clean)}")


def _ran_proj_case(name, x, k, l, q, seed, store_x=True, store_result=True, scaled_alpha=None,
                   x_seed=None, x_kind=None):
    """ran_proj (or ran_proj_scal with a fixed α) on a Generator(seed); Ω = first draw."""
    n = x.shape[0]
    omega = np.random.default_rng(seed).standard_normal((n, k + l))
    rng = np.random.default_rng(seed)
    if scaled_alpha is None:
        rep = psdcone.ran_proj(x, RangeParams(k=k, l=l, q=q), rng, return_factors=True,
                               collect_diagnostics=True)
    else:
        rep = psdcone.ran_proj_scal(x, RangeParams(k=k, l=l, q=q), scaled_alpha, rng,
                                    return_factors=True, collect_diagnostics=True)
    w, d = rep.factors
    _save(name,
          x=x if store_x else None,
          x_seed=x_seed, x_kind=x_kind,
          x_checksum=np.array([float(np.sum(x)), float(np.linalg.norm(x))]),
          omega=omega, k=k, l=l, q=q, seed=seed,
          alpha=scaled_alpha if scaled_alpha is not None else 0.0,
          result=rep.result if store_result else None,
          result_checksum=np.array([float(np.sum(rep.result)), float(np.linalg.norm(rep.result))]),
          w=w, d=d, effective_rank=rep.effective_rank, basis_width=rep.basis_width,
          residual_frob=rep.residual_frob)


def main():
    # --- SPEC known answers ---------------------------------
    x3 = np.diag([-3.0, -2.0, 1.0])
    _ran_proj_case("spec_counterexample_full", x3, 1, 2, 0, seed=0)
    _ran_proj_case("spec_scal_alpha3_full", x3, 1, 2, 0, seed=0, scaled_alpha=3.0)
    _ran_proj_case("spec_scal_alpha3_k1", x3, 1, 0, 1, seed=5, scaled_alpha=3.0)

    rng = np.random.default_rng(11)
    z = rng.standard_normal((40, 3))
    _ran_proj_case("spec_psd_fixed_point", z @ z.T, 4, 2, 0, seed=3)

    u = np.random.default_rng(12).standard_normal(50)
    u /= np.linalg.norm(u)
    _ran_proj_case("rank1_truncation", np.outer(u, u), 3, 2, 0, seed=4)
    _ran_proj_case("zero_matrix", np.zeros((20, 20)), 2, 2, 1, seed=5)
    _ran_proj_case("n1_positive", np.array([[2.5]]), 1, 0, 1, seed=6)
    _ran_proj_case("n1_negative", np.array([[-1.0]]), 1, 0, 0, seed=7)

    # --- random Wigner, every q regime (q>=2 stabilised) ---------------------
    for q in (0, 1, 2, 3):
        _ran_proj_case(f"wigner64_q{q}", orc.wigner(64, seed=20 + q), 8, 4, q, seed=30 + q)
    _ran_proj_case("wigner200_k37_q1", orc.wigner(200, seed=40), 37, 5, 1, seed=41,
                   store_x=False, store_result=False, x_seed=40, x_kind="wigner")

    # --- C3-shaped (ill-conditioned unstabilised q=1) at reduced n ------------
    _ran_proj_case("c3like_n512_q1", orc.c3_matrix(512, seed=50, rank=40), 48, 8, 1, seed=51,
                   store_x=False, store_result=False, x_seed=50, x_kind="c3r40")

    # --- within-tolerance asymmetry: exercises the Xᵀ multiply (sketch.py:79) -
    xa = orc.wigner(96, seed=60)
    xa = xa + 2e-12 * np.random.default_rng(61).standard_normal(xa.shape)
    _ran_proj_case("nearsym96_q1", xa, 10, 6, 1, seed=62)

    # --- scaled, fixed α (experiments.py:110 style) ---------------------------
    _ran_proj_case("wigner128_scal", orc.wigner(128, seed=70), 12, 6, 1, seed=71, scaled_alpha=0.9)

    # --- scaled with α estimated inside project() (draw order: v1, v2, Ω) -----
    for name, x, k, l, q, seed, sf in (
        ("project_scaled_est_wigner80", orc.wigner(80, seed=80) - 0.2 * np.eye(80), 10, 5, 1, 81, 1.0),
        ("project_scaled_half_wigner80", orc.wigner(80, seed=82), 10, 5, 2, 83, 0.5),
    ):
        n = x.shape[0]
        g = np.random.default_rng(seed)
        v1 = g.standard_normal(n)
        v2 = g.standard_normal(n)
        omega = g.standard_normal((n, k + l))
        cfg = ProjectorConfig(method="scaled_randomized", params=RangeParams(k=k, l=l, q=q),
                              power_N=10, scale_factor=sf, return_factors=True)
        rep = psdcone.project(x, cfg, seed)
        w, d = rep.factors
        _save(name, x=x, omega=omega, v1=v1, v2=v2, k=k, l=l, q=q, seed=seed, power_n=10,
              scale_factor=sf, alpha_used=rep.alpha_used, fallback=rep.fallback,
              result=rep.result, w=w, d=d, effective_rank=rep.effective_rank,
              basis_width=rep.basis_width)

    # --- AlphaTooSmall fallback (projection.py:214-221) -----------------------
    zz = np.random.default_rng(90).standard_normal((30, 4))
    xp = zz @ zz.T
    cfg = ProjectorConfig(method="scaled_randomized", params=RangeParams(k=5, l=2, q=1),
                          alpha_override=1e-14, return_factors=True)
    omega = np.random.default_rng(91).standard_normal((30, 7))
    rep = psdcone.project(xp, cfg, 91)
    _save("project_alpha_fallback", x=xp, omega=omega, k=5, l=2, q=1, seed=91,
          alpha_override=1e-14, alpha_used=rep.alpha_used, fallback=rep.fallback,
          result=rep.result, effective_rank=rep.effective_rank, basis_width=rep.basis_width)

    # --- power iteration / min-eig known answers ------------
    pis = []
    for name, x, nit, seed in (
        ("diag51", np.diag([5.0, 1.0]), 10, 1),
        ("zero", np.zeros((4, 4)), 10, 2),
        ("wigner300", orc.wigner(300, seed=3), 10, 4),
    ):
        v0 = np.random.default_rng(seed).standard_normal(x.shape[0])
        val = psdcone.power_iteration(x, nit, np.random.default_rng(seed))
        pis.append((name, x, nit, v0, val))
    for name, x, nit, v0, val in pis:
        big = x.shape[0] > 100
        _save(f"power_iteration_{name}", x=None if big else x, x_kind="wigner" if big else None,
              x_seed=3 if big else None, n=x.shape[0], n_iter=nit, v0=v0, value=val)
    for name, x, seed in (
        ("diag_m3m21", np.diag([-3.0, -2.0, 1.0]), 1),
        ("diag_123", np.diag([1.0, 2.0, 3.0]), 2),
        ("minus_eye2", -np.eye(2), 3),
        ("wigner300", orc.wigner(300, seed=5), 6),
    ):
        g = np.random.default_rng(seed)
        v1 = g.standard_normal(x.shape[0])
        v2 = g.standard_normal(x.shape[0])
        val = psdcone.min_eig_magnitude(x, 10, np.random.default_rng(seed))
        big = x.shape[0] > 100
        _save(f"min_eig_{name}", x=None if big else x, x_kind="wigner" if big else None,
              x_seed=5 if big else None, n=x.shape[0], n_iter=10, v1=v1, v2=v2, value=val)

    # --- eigh convention (symmetric.py:68-86) ---------------------------------
    te = orc.wigner(50, seed=95)
    dec = psdcone.eigh(te)
    _save("eigh_wigner50", x=te, values=dec.values, vectors=dec.vectors)

    # --- BASELINE config 1 (n=1000): X regenerated from seed, factors stored --
    x1 = orc.c1_matrix(seed=0)
    _ran_proj_case("config1_ran_proj", x1, 40, 10, 2, seed=1, store_x=False, store_result=False,
                   x_seed=0, x_kind="c1")
    g = np.random.default_rng(2)
    v1 = g.standard_normal(1000)
    v2 = g.standard_normal(1000)
    omega = g.standard_normal((1000, 50))
    cfg = ProjectorConfig(method="scaled_randomized", params=RangeParams(k=40, l=10, q=2),
                          power_N=10, return_factors=True)
    rep = psdcone.project(x1, cfg, 2)
    w, d = rep.factors
    _save("config1_project_scaled", x_seed=0, x_kind="c1",
          x_checksum=np.array([float(np.sum(x1)), float(np.linalg.norm(x1))]),
          omega=omega, v1=v1, v2=v2, k=40, l=10, q=2, seed=2, power_n=10, scale_factor=1.0,
          alpha_used=rep.alpha_used, fallback=rep.fallback, w=w, d=d,
          result_checksum=np.array([float(np.sum(rep.result)), float(np.linalg.norm(rep.result))]),
          effective_rank=rep.effective_rank, basis_width=rep.basis_width)


def solver_cases():
    """Reference solve() (sdls.py:164-265) on small dense SDLS instances."""
    from oracle import sdls_oracle as so
    for name, method, n, m, k, l, q, refresh in (
        ("sdls_randomized", "randomized", 40, 12, 8, 4, 1, 1),
        ("sdls_scaled", "scaled_randomized", 36, 10, 6, 4, 1, 3),
    ):
        sp = so.config5_instance(n, m, nnz_per=4, seed=123 + n)
        dense = np.zeros((m, n, n))
        np.add.at(dense, (sp.con, sp.rows, sp.cols), sp.vals)
        beta = so.lipschitz_beta(sp)
        problem = psdcone.SdlsProblem(sp.c, 1.0, list(zip(dense, sp.b)))
        cfg = ProjectorConfig(method=method, params=RangeParams(k=k, l=l, q=q), power_N=10)
        rep = psdcone.solve(problem, cfg, beta=beta, epsilon=1e-14, max_iter=25, rng=7,
                            alpha_refresh=refresh, keep_trajectory=True)
        _save(name, c=sp.c, con=sp.con, rows=sp.rows, cols=sp.cols, vals=sp.vals, b=sp.b,
              n=n, m=m, k=k, l=l, q=q, beta=beta, seed=7, alpha_refresh=refresh,
              method=method, y_final=rep.y_final,
              grad_norms=np.array([t.grad_norm for t in rep.trajectory]),
              x_solution=rep.x_solution, objective=rep.objective,
              iterations=rep.iterations, exact_residual=rep.exact_feasibility_residual)


def solver_dense_cases():
    """Reference solve() with the exact projector (its default, sdls.py:187) and
    the polar projector: no sketch RNG, dense X₊ every iteration."""
    from oracle import sdls_oracle as so
    for name, method, n, m in (("sdls_exact", "exact", 32, 10), ("sdls_polar", "polar", 28, 8)):
        sp = so.config5_instance(n, m, nnz_per=4, seed=321 + n)
        dense = np.zeros((m, n, n))
        np.add.at(dense, (sp.con, sp.rows, sp.cols), sp.vals)
        beta = so.lipschitz_beta(sp)
        problem = psdcone.SdlsProblem(sp.c, 1.0, list(zip(dense, sp.b)))
        cfg = None if method == "exact" else ProjectorConfig(method=method)
        rep = psdcone.solve(problem, cfg, beta=beta, epsilon=1e-14, max_iter=20, rng=8,
                            keep_trajectory=True)
        _save(name, c=sp.c, con=sp.con, rows=sp.rows, cols=sp.cols, vals=sp.vals, b=sp.b,
              n=n, m=m, beta=beta, seed=8, method=method, y_final=rep.y_final,
              grad_norms=np.array([t.grad_norm for t in rep.trajectory]),
              x_solution=rep.x_solution, objective=rep.objective,
              iterations=rep.iterations, feasibility=rep.feasibility_residual)


def sweep_cases():
    """Reference projection_error_sweep (experiments.py:78-137) and bounds (bounds.py)."""
    from psdcone import bounds as rb
    from psdcone import experiments as rx
    codes = {"randomized": 0, "scaled_randomized": 1}
    for name, n, l, q, k_grid, trials, seed in (
        ("sweep_fourblock_q0", 64, 4, 0, (4, 8, 16), 2, 5),
        ("sweep_fourblock_q1", 64, 4, 1, (8, 12), 2, 9),
    ):
        rows = rx.projection_error_sweep(n, rx.FOUR_BLOCK_BETAS, l, q, k_grid, trials, seed)
        x = rx.four_block_matrix(n, rx.FOUR_BLOCK_BETAS, np.random.default_rng(seed))
        _save(name, n=n, l=l, q=q, k_grid=np.array(k_grid), trials=trials, seed=seed, x=x,
              k=np.array([r.k for r in rows]), method=np.array([codes[r.method] for r in rows]),
              mean_frob=np.array([r.mean_frob_error for r in rows]),
              mean_spec=np.array([r.mean_spectral_error for r in rows]),
              frob_bound=np.array([np.nan if r.frob_bound is None else r.frob_bound for r in rows]),
              spec_bound=np.array([r.spectral_bound for r in rows]))
    # bounds on a generic spectrum (descending, mixed signs)
    ev = np.sort(np.random.default_rng(3).standard_normal(40) * np.geomspace(10, 0.01, 40))[::-1]
    spec = rb.SpectrumSummary.from_eigenvalues(ev)
    vals = []
    for k, l, q, alpha in ((3, 2, 0, 0.5), (10, 5, 0, 2.0), (10, 5, 1, 2.0), (20, 8, 2, 0.1)):
        p = rb.BoundParams(k=k, l=l, q=q)
        vals.append([k, l, q, alpha, rb.eps1(spec.sigmas, k, l), rb.eps2(spec.sigmas[k], k, l, q, 40),
                     rb.frob_bound_unscaled(spec, p) if q == 0 else np.nan,
                     rb.spectral_bound_unscaled(spec, p),
                     rb.frob_bound_scaled(spec, p, alpha) if q == 0 else np.nan,
                     rb.spectral_bound_scaled(spec, p, alpha)])
    _save("bounds_generic", eigenvalues=ev, table=np.array(vals))


if __name__ == "__main__":
    import sys as _sys
    if "--sweep-only" in _sys.argv:
        sweep_cases()
    elif "--dense-solver-only" in _sys.argv:
        solver_dense_cases()
    else:
        main()
        solver_cases()
        solver_dense_cases()
        sweep_cases()
