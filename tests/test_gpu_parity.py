"""GPU parity: libpsdproj.so (through the reference-shaped API and the C ABI)
against the reference's golden outputs and the CPU oracle on identical X and Ω.

Tolerance (BASELINE.json north_star): relative Frobenius error ≤ 1e-10 in
FP64.  Integer outputs (effective_rank, basis_width, fallback) must be equal.
"""

import numpy as np
import pytest

from oracle import psd_oracle as orc
from tests import golden_io as gio

pytestmark = pytest.mark.gpu

TOL = 1e-10

RAN_CASES = [n for n in gio.names() if "w" in np.load(f"{gio.GOLDEN}/{n}.npz").files
             and not n.startswith(("project_", "config1_project"))]


def _rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


@pytest.fixture(scope="module")
def ours():
    import paper_2410_19208_b200 as m
    m._native.load_library()
    return m


@pytest.fixture(params=["auto", "int8"])
def engine(request, ours):
    """FP64 product engine: "auto" (DMMA below n = 3072, INT8 emulation above) and
    "int8" forced at every size, so the golden parity runs on both engines."""
    prev = ours.set_fp64_engine(request.param)
    yield request.param
    ours.set_fp64_engine(prev)


@pytest.mark.parametrize("name", RAN_CASES)
def test_ran_proj_golden(ours, engine, name):
    d = gio.load(name)
    params = ours.RangeParams(k=int(d["k"]), l=int(d["l"]), q=int(d["q"]))
    alpha = float(d["alpha"])
    if alpha > 0:
        rep = ours.ran_proj_scal(d["x"], params, alpha, None, collect_diagnostics=True,
                                 return_factors=True, omega=d["omega"])
    else:
        rep = ours.ran_proj(d["x"], params, None, collect_diagnostics=True, return_factors=True,
                            omega=d["omega"])
    ref = gio.golden_result(d)
    assert rep.basis_width == int(d["basis_width"])
    assert rep.effective_rank == int(d["effective_rank"])
    assert isinstance(rep.result, np.ndarray) and rep.result.shape == ref.shape
    assert _rel(rep.result, ref) <= TOL, _rel(rep.result, ref)
    np.testing.assert_array_equal(rep.result, rep.result.T)      # mirrored store: exact symmetry
    w, dd = rep.factors
    assert w.shape == (ref.shape[0], rep.effective_rank)
    np.testing.assert_allclose(np.sort(dd), np.sort(d["d"]), rtol=1e-9, atol=1e-12 * max(1, abs(d["d"]).max(initial=0)))
    if "residual_frob" in d:
        assert rep.residual_frob == pytest.approx(float(d["residual_frob"]), rel=1e-6, abs=1e-9)


@pytest.mark.parametrize("name", gio.names("project_") + ["config1_project_scaled"])
def test_project_scaled_golden(ours, engine, name):
    d = gio.load(name)
    params = ours.RangeParams(k=int(d["k"]), l=int(d["l"]), q=int(d["q"]))
    if "alpha_override" in d:
        cfg = ours.ProjectorConfig(method="scaled_randomized", params=params,
                                   alpha_override=float(d["alpha_override"]))
    else:
        cfg = ours.ProjectorConfig(method="scaled_randomized", params=params,
                                   power_N=int(d["power_n"]), scale_factor=float(d["scale_factor"]))
    # same seed → same numpy stream → same v1, v2, Ω draw order as the reference
    rep = ours.project(d["x"], cfg, int(d["seed"]))
    assert rep.fallback == bool(d["fallback"])
    assert rep.alpha_used == pytest.approx(float(d["alpha_used"]), rel=1e-11)
    assert rep.effective_rank == int(d["effective_rank"])
    assert _rel(rep.result, gio.golden_result(d)) <= TOL


@pytest.mark.parametrize("name", gio.names("power_iteration_"))
def test_power_iteration_golden(ours, name):
    d = gio.load(name)
    val = ours.power_iteration(d["x"], int(d["n_iter"]), None, v0=d["v0"])
    assert val == pytest.approx(float(d["value"]), rel=1e-12, abs=0.0)


@pytest.mark.parametrize("name", gio.names("min_eig_"))
def test_min_eig_golden(ours, name):
    d = gio.load(name)
    val = ours.min_eig_magnitude(d["x"], int(d["n_iter"]), None, v1=d["v1"], v2=d["v2"])
    assert val == pytest.approx(float(d["value"]), rel=1e-10, abs=1e-13)


def test_eigh_golden(ours):
    d = gio.load("eigh_wigner50")
    dec = ours.eigh(d["x"])
    np.testing.assert_allclose(dec.values, d["values"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(dec.vectors, d["vectors"], rtol=0, atol=1e-10)


@pytest.mark.parametrize("n,k,l,q,seed", [(300, 20, 6, 0, 1), (513, 40, 9, 1, 2), (777, 30, 10, 3, 3)])
def test_ran_proj_vs_oracle_random_shapes(ours, engine, n, k, l, q, seed):
    x = orc.wigner(n, seed=seed)
    om = np.random.default_rng(seed + 100).standard_normal((n, k + l))
    ref = orc.ran_proj(x, k, l, q, omega=om)
    rep = ours.ran_proj(x, ours.RangeParams(k=k, l=l, q=q), None, omega=om)
    assert rep.effective_rank == ref.effective_rank
    assert _rel(rep.result, ref.result) <= TOL


@pytest.mark.parametrize("n", [2048, 4096])
def test_config3_shape_reduced_n(ours, engine, n):
    """C3 spectrum (rank-200 ± parts + 1e-3 Wigner), k=256, p=16, q=1: the
    unstabilised, κ(Y)≈1e8 case that stresses the CholeskyQR path."""
    x = orc.c3_matrix(n, seed=7)
    om = np.random.default_rng(8).standard_normal((n, 272))
    ref = orc.ran_proj(x, 256, 16, 1, omega=om)
    rep = ours.ran_proj(x, ours.RangeParams(k=256, l=16, q=1), None, omega=om)
    assert rep.basis_width == ref.basis_width
    assert rep.effective_rank == ref.effective_rank
    assert _rel(rep.result, ref.result) <= TOL, _rel(rep.result, ref.result)


def test_config2_full_size(ours):
    """BASELINE config 2 at full size: n=8192 Wigner, k=128, p=16, q=2."""
    x = orc.wigner(8192, seed=2)
    om = np.random.default_rng(3).standard_normal((8192, 144))
    ref = orc.ran_proj(x, 128, 16, 2, omega=om)
    rep = ours.ran_proj(x, ours.RangeParams(k=128, l=16, q=2), None, omega=om)
    assert rep.effective_rank == ref.effective_rank
    assert _rel(rep.result, ref.result) <= TOL


def test_range_finder_rectangular(ours):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((300, 180))
    om = rng.standard_normal((180, 25))
    ref_q, _, _, _ = orc.range_finder(x, 20, 5, 2, omega=om)
    q = ours.range_finder(x, ours.RangeParams(k=20, l=5, q=2), None, omega=om)
    assert q.shape == ref_q.shape
    # same span: projectors agree
    assert _rel(q @ q.T, ref_q @ ref_q.T) <= 1e-10
    assert ours.orthonormality_defect(q) <= 1e-12 * 25


def test_torch_in_torch_out(ours):
    import torch
    x = orc.wigner(500, seed=9)
    om = np.random.default_rng(10).standard_normal((500, 30))
    xt = torch.from_numpy(x).cuda()
    rep = ours.ran_proj(xt, ours.RangeParams(k=24, l=6, q=1), None, omega=torch.from_numpy(om).cuda())
    assert isinstance(rep.result, torch.Tensor) and rep.result.is_cuda
    ref = orc.ran_proj(x, 24, 6, 1, omega=om)
    assert _rel(rep.result.cpu().numpy(), ref.result) <= TOL


def test_errors_match_reference(ours):
    with pytest.raises(ours.AsymmetricMatrixError):
        ours.ran_proj(np.array([[1.0, 2.0], [0.0, 1.0]]), ours.RangeParams(k=1), None, omega=np.ones((2, 1)))
    with pytest.raises(ours.NonSquareError):
        ours.ran_proj(np.ones((3, 4)), ours.RangeParams(k=1), None)
    with pytest.raises(ours.InvalidParams):
        ours.ran_proj(np.eye(3), ours.RangeParams(k=3, l=1), np.random.default_rng(0))
    with pytest.raises(ours.AlphaTooSmall):
        ours.ran_proj_scal(np.eye(3), ours.RangeParams(k=1, l=1), 1e-13, np.random.default_rng(0))
    u = np.random.default_rng(1).standard_normal(30)
    with pytest.raises(ours.RankDeficientSample):
        ours.range_finder(np.outer(u, u), ours.RangeParams(k=3, l=2), np.random.default_rng(2),
                          strict=True)


def test_rng_draw_order_matches_reference(ours):
    """project(randomized, seed) consumes Ω as the first draw of default_rng(seed)."""
    x = orc.wigner(120, seed=11)
    rep = ours.project(x, ours.ProjectorConfig(method="randomized", params=ours.RangeParams(k=10, l=5, q=1)), 77)
    om = np.random.default_rng(77).standard_normal((120, 15))
    ref = orc.ran_proj(x, 10, 5, 1, omega=om)
    assert _rel(rep.result, ref.result) <= TOL


def test_exact_projection(ours):
    x = orc.wigner(100, seed=12)
    rep = ours.project(x, ours.ProjectorConfig(method="exact"))
    ref = orc.exact_psd_projection(x)
    assert _rel(rep.result, ref) <= 1e-10
    rep2 = ours.project(x, ours.ProjectorConfig(method="polar"))
    assert _rel(rep2.result, ref) <= 1e-8


@pytest.mark.parametrize("n,k,l,q,alpha", [(1024, 40, 8, 1, 0.0), (777, 30, 9, 2, 0.0), (900, 24, 8, 1, 0.6)])
def test_sharded_single_rank_kernel_ops(ours, n, k, l, q, alpha):
    """The row-sharded driver on one rank with the real kernels."""
    import torch
    from paper_2410_19208_b200.sharded import KernelOps, sharded_ran_proj
    x = orc.wigner(n, seed=21)
    om = np.random.default_rng(22).standard_normal((n, k + l))
    ref = orc.ran_proj_scal(x, k, l, q, alpha, omega=om) if alpha > 0 else orc.ran_proj(x, k, l, q, omega=om)
    for engine in ("int8", "dmma"):
        prev = ours.set_fp64_engine(engine)
        try:
            ops = KernelOps("cuda")
            rep = sharded_ran_proj(torch.from_numpy(x).cuda(), 0, n, torch.from_numpy(om).cuda(),
                                   ours.RangeParams(k=k, l=l, q=q), alpha=alpha, ops=ops)
        finally:
            ours.set_fp64_engine(prev)
        assert (ops.int8_products > 0) == (engine == "int8")
        assert rep.effective_rank == ref.effective_rank
        res = rep.result_rows.cpu().numpy()
        assert np.array_equal(res, res.T)
        assert _rel(res, ref.result) <= TOL


def test_c4_row_blocks_assemble_symmetric(ours):
    """Config-4 generator: row blocks built independently are bitwise symmetric together."""
    import torch
    from paper_2410_19208_b200 import workloads
    n = 2048
    a = workloads.c4_rows(n, 0, 1000, seed=3)
    b = workloads.c4_rows(n, 1000, n, seed=3, chunk_rows=300)
    x = torch.cat([a, b], 0)
    assert torch.equal(x, x.T)
    full = workloads.c4_rows(n, 0, n, seed=3)
    assert torch.equal(full, x)


@pytest.mark.parametrize("name", ["sdls_randomized", "sdls_scaled"])
def test_solver_loop_matches_reference(ours, name):
    """Alg. 6 (sdls.py:164-265) on the device vs the reference's own trajectory."""
    d = gio.load(name)
    prob = ours.SparseSdlsProblem(d["c"], 1.0, d["con"], d["rows"], d["cols"], d["vals"], d["b"])
    cfg = ours.ProjectorConfig(method=str(d["method"]),
                               params=ours.RangeParams(k=int(d["k"]), l=int(d["l"]), q=int(d["q"])),
                               power_N=10)
    rep = ours.solve(prob, cfg, beta=float(d["beta"]), epsilon=1e-14, max_iter=25,
                     rng=int(d["seed"]), alpha_refresh=int(d["alpha_refresh"]), keep_trajectory=True)
    assert rep.iterations == int(d["iterations"])
    np.testing.assert_allclose([t.grad_norm for t in rep.trajectory], d["grad_norms"], rtol=1e-8)
    np.testing.assert_allclose(rep.y_final, d["y_final"], rtol=1e-8, atol=1e-11)
    assert _rel(rep.x_solution, d["x_solution"]) <= 1e-9
    assert rep.objective == pytest.approx(float(d["objective"]), rel=1e-8)
    assert rep.exact_feasibility_residual == pytest.approx(float(d["exact_residual"]), rel=1e-6)
