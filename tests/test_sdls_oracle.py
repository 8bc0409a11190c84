"""The solver-loop oracle (oracle/sdls_oracle.py) against the reference's own
solve() trajectories (tests/golden/sdls_*.npz), for the dense stack and for the
sparse-COO rebinding used at config-5 scale."""

import numpy as np
import pytest

from oracle import sdls_oracle as so
from tests import golden_io as gio


def _problems(d):
    n, m = int(d["n"]), int(d["m"])
    sp = so.SparseProblem(d["c"], 1.0, d["con"], d["rows"], d["cols"], d["vals"], d["b"])
    dense = np.zeros((m, n, n))
    np.add.at(dense, (d["con"], d["rows"], d["cols"]), d["vals"])
    return so.DenseProblem(d["c"], 1.0, dense, d["b"]), sp


@pytest.mark.parametrize("name", ["sdls_randomized", "sdls_scaled"])
@pytest.mark.parametrize("kind", ["dense", "sparse"])
def test_solver_oracle_matches_reference(name, kind):
    d = gio.load(name)
    dense, sparse = _problems(d)
    prob = dense if kind == "dense" else sparse
    rep = so.solve(prob, str(d["method"]), int(d["k"]), int(d["l"]), int(d["q"]),
                   beta=float(d["beta"]), epsilon=1e-14, max_iter=25, rng=int(d["seed"]),
                   alpha_refresh=int(d["alpha_refresh"]))
    assert rep.iterations == int(d["iterations"])
    np.testing.assert_allclose(rep.trajectory, d["grad_norms"], rtol=1e-9)
    np.testing.assert_allclose(rep.y_final, d["y_final"], rtol=1e-9, atol=1e-12)
    err = np.linalg.norm(rep.x_solution - d["x_solution"]) / np.linalg.norm(d["x_solution"])
    assert err < 1e-9
    assert rep.objective == pytest.approx(float(d["objective"]), rel=1e-9)
    assert rep.exact_feasibility_residual == pytest.approx(float(d["exact_residual"]), rel=1e-8)


@pytest.mark.parametrize("name", ["sdls_exact", "sdls_polar"])
def test_dense_projector_solver_oracle_matches_reference(name):
    """The exact (reference default) and polar projectors inside solve()."""
    d = gio.load(name)
    dense, sparse = _problems(d)
    for prob in (dense, sparse):
        rep = so.solve(prob, str(d["method"]), 1, 0, 0, beta=float(d["beta"]), epsilon=1e-14,
                       max_iter=20, rng=int(d["seed"]))
        assert rep.iterations == int(d["iterations"])
        np.testing.assert_allclose(rep.trajectory, d["grad_norms"], rtol=1e-9)
        np.testing.assert_allclose(rep.y_final, d["y_final"], rtol=1e-9, atol=1e-12)
        err = np.linalg.norm(rep.x_solution - d["x_solution"]) / np.linalg.norm(d["x_solution"])
        assert err < 1e-9
        assert rep.exact_feasibility_residual is None


def test_config5_instance_shapes():
    p = so.config5_instance(64, 30, seed=1)
    assert p.con.size == 30 * 8 and p.b.shape == (30,)
    x = p.assemble(np.ones(30))
    np.testing.assert_array_equal(x, x.T)
    beta = so.lipschitz_beta(p)
    assert 0 < beta < 1


def test_product_config5_generator_matches_the_oracle_instance():
    """bench.py's own arm builds config 5 with the package's generator
    (workloads.c5_problem / c5_step_size); the CPU arm solves the oracle's
    SparseProblem of the same triplets — both must be the same instance."""
    from oracle import sdls_oracle as so
    from paper_2410_19208_b200 import workloads
    ours = workloads.c5_problem(192, 300, nnz_per=4, seed=5)
    ref = so.config5_instance(192, 300, nnz_per=4, seed=5)
    for name in ("c", "con", "rows", "cols", "vals", "b"):
        assert np.array_equal(getattr(ours, name), getattr(ref, name)), name
    assert ours.rho == ref.rho
    assert np.all(ours.rows != ours.cols)
    assert workloads.c5_step_size(ours, iters=20) == so.lipschitz_beta(ref, iters=20)
