"""Command-line front end (``harness_cli``; the reference
declares ``psdcone = "psdcone.cli:main"`` at pkg/pyproject.toml:15-16 but ships
no module).  Every numeric step runs on the GPU through this package.

    python -m paper_2410_19208_b200 project --input X.mtx --method randomized \
        --k 40 --l 10 --q 2 --seed 7 --output Xp.mtx [--report rep.json]
    python -m paper_2410_19208_b200 solve --problem p.json --proj randomized \
        --k 32 --l 10 --q 1 --beta 0.02 --epsilon 1e-8 --max-iter 300 --seed 1 --report s.json
    python -m paper_2410_19208_b200 fig4 --n 1000 --betas 3,1,6,2 --l 5 --q 2 \
        --k-grid 100,200 --trials 2 --seed 0 --out fig4.csv

Exit codes: 0 success, 2 validation / I-O failure, 3 numerical
failure.  Failures print one JSON object {"error": <class>, "message": ...} on
stderr.
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import sys

from . import errors

_METHOD = {"exact": "exact", "polar": "polar", "randomized": "randomized", "scaled": "scaled_randomized"}
# numerical failures → exit 3; everything else a PsdconeError reports is validation → exit 2
_NUMERICAL = ("ConvergenceFailure", "RankDeficientSample", "AlphaTooSmall")


class _ArgError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):   # argparse exits 2 by itself; route through the JSON error channel
        raise _ArgError(message)


def _csv_floats(text, what):
    try:
        return [float(t) for t in text.split(",") if t.strip()]
    except ValueError:
        raise errors.error("InvalidParams", f"{what}: expected comma-separated numbers, got {text!r}")


def _jsonable(v):
    if isinstance(v, float) and not math.isfinite(v):
        return None if math.isnan(v) else ("inf" if v > 0 else "-inf")
    if hasattr(v, "tolist"):
        return v.tolist()
    return v


def _params(a):
    from .sketch import RangeParams
    return RangeParams(k=a.k, l=a.l, q=a.q, seed=a.seed)


def cmd_project(a):
    """cli_project: read X, project, write X̂₊ and a JSON report."""
    from .matrix_io import read_matrix_market, write_matrix_market
    from .projection import ProjectorConfig, project
    x = read_matrix_market(a.input)
    method = _METHOD[a.method]
    params = _params(a) if method in ("randomized", "scaled_randomized") else None
    if params is not None and params.width > min(x.shape):
        raise errors.error("InvalidParams", f"k+l exceeds dimension ({params.width} > {min(x.shape)})")
    cfg = ProjectorConfig(method=method, params=params, power_N=a.N, alpha_override=a.alpha,
                          collect_diagnostics=a.diagnostics, dtype=a.dtype)
    rep = project(x, cfg, a.seed)
    write_matrix_market(a.output, rep.result, fmt="array")
    doc = {"method": rep.method, "effective_rank": rep.effective_rank, "alpha_used": rep.alpha_used,
           "residual_frob": rep.residual_frob, "fallback": rep.fallback, "basis_width": rep.basis_width,
           "n": int(x.shape[0]), "seed": a.seed, "output": a.output}
    if a.report:
        with open(a.report, "w") as fh:
            json.dump({k: _jsonable(v) for k, v in doc.items()}, fh, indent=1, sort_keys=True)
    return 0


def cmd_solve(a):
    """cli_solve: dual ascent (Alg. 6) on a JSON problem file."""
    from .matrix_io import read_sdls_problem
    from .projection import ProjectorConfig
    from .sdls import SparseSdlsProblem, solve
    prob = read_sdls_problem(a.problem)
    if a.rho_override is not None:
        prob = SparseSdlsProblem(prob.c, a.rho_override, prob.con, prob.rows, prob.cols, prob.vals, prob.b)
    method = _METHOD[a.proj]
    if method not in ("randomized", "scaled_randomized"):
        raise errors.error("InvalidParams", "the device solver runs --proj randomized or scaled")
    cfg = ProjectorConfig(method=method, params=_params(a), power_N=a.N)
    rep = solve(prob, cfg, beta=a.beta, epsilon=a.epsilon, max_iter=a.max_iter, rng=a.seed)
    doc = {"y_final": rep.y_final, "iterations": rep.iterations, "grad_norm_final": rep.grad_norm_final,
           "feasibility_residual": rep.feasibility_residual, "objective": rep.objective,
           "projection_method": rep.projection_method, "converged": rep.converged,
           "exact_feasibility_residual": rep.exact_feasibility_residual, "n": prob.n, "m": prob.m,
           "seed": a.seed}
    text = json.dumps({k: _jsonable(v) for k, v in doc.items()}, indent=1, sort_keys=True)
    if a.report:
        with open(a.report, "w") as fh:
            fh.write(text)
    else:
        print(text)
    return 0


def cmd_fig4(a):
    """cli_bench_fig4: projection-error sweep → CSV."""
    from .experiments import projection_error_sweep
    betas = _csv_floats(a.betas, "--betas")
    if len(betas) != 4:
        raise errors.error("InvalidParams", f"--betas needs four values, got {betas}")
    grid = [int(k) for k in _csv_floats(a.k_grid, "--k-grid")]
    rows = projection_error_sweep(a.n, tuple(betas), a.l, a.q, grid, a.trials, a.seed)
    with open(a.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["k", "method", "mean_frob_error", "mean_spectral_error", "frob_bound", "spectral_bound"])
        for r in rows:
            w.writerow([r.k, r.method, repr(r.mean_frob_error), repr(r.mean_spectral_error),
                        "" if r.frob_bound is None else repr(r.frob_bound),
                        "" if r.spectral_bound is None else repr(r.spectral_bound)])
    return 0


def build_parser():
    p = _Parser(prog="python -m paper_2410_19208_b200", description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True)

    def sketch_flags(sp, method_flag, choices):
        sp.add_argument(method_flag, choices=choices, required=True)
        sp.add_argument("--k", type=int, default=10)
        sp.add_argument("--l", type=int, default=10)
        sp.add_argument("--q", type=int, default=0)
        sp.add_argument("--N", type=int, default=10, help="power iterations of the alpha estimate")
        sp.add_argument("--seed", type=int, default=0)

    sp = sub.add_parser("project", help="project a Matrix Market matrix onto the PSD cone")
    sp.add_argument("--input", required=True)
    sp.add_argument("--output", required=True)
    sketch_flags(sp, "--method", sorted(_METHOD))
    sp.add_argument("--alpha", type=float, default=None, help="alpha override of the scaled method")
    sp.add_argument("--diagnostics", action="store_true")
    sp.add_argument("--dtype", choices=["fp64", "fp32"], default="fp64")
    sp.add_argument("--report", default=None)
    sp.set_defaults(fn=cmd_project)

    sp = sub.add_parser("solve", help="dual ascent on a JSON SDLS problem")
    sp.add_argument("--problem", required=True)
    sketch_flags(sp, "--proj", sorted(_METHOD))
    sp.add_argument("--rho-override", type=float, default=None)
    sp.add_argument("--beta", type=float, default=0.5)
    sp.add_argument("--epsilon", type=float, default=1e-8)
    sp.add_argument("--max-iter", type=int, default=100)
    sp.add_argument("--report", default=None)
    sp.set_defaults(fn=cmd_solve)

    sp = sub.add_parser("fig4", help="Fig. 4 projection-error sweep (CSV)")
    sp.add_argument("--n", type=int, default=1000)
    sp.add_argument("--betas", default="3,1,6,2", help="four-block spectrum betas (experiments.py:31)")
    sp.add_argument("--l", type=int, default=5)
    sp.add_argument("--q", type=int, default=2)
    sp.add_argument("--k-grid", default="100,200,300")
    sp.add_argument("--trials", type=int, default=1)
    sp.add_argument("--seed", type=int, default=0)
    sp.add_argument("--out", required=True)
    sp.set_defaults(fn=cmd_fig4)
    return p


def _fail(kind, message, code):
    print(json.dumps({"error": kind, "message": str(message)}), file=sys.stderr)
    return code


def main(argv=None):
    try:
        a = build_parser().parse_args(argv)
    except _ArgError as exc:
        return _fail("InvalidParams", exc, 2)
    try:
        return a.fn(a)
    except errors.PsdconeError as exc:
        kind = type(exc).__name__
        return _fail(kind, exc, 3 if kind in _NUMERICAL else 2)
    except (OSError, ValueError) as exc:
        return _fail(type(exc).__name__, exc, 2)


if __name__ == "__main__":
    sys.exit(main())
