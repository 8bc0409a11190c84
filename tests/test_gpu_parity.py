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


@pytest.mark.slow
@pytest.mark.parametrize("seed", [1, 2])
def test_config3_full_size_fp64(ours, seed):
    """BASELINE config 3 at FULL size (n = 32768, k = 256, p = 16, q = 1) on the default
    engines (INT8-emulated FP64 products + INT8 reconstruction) against the CPU oracle
    on the identical X and Ω; the whole n×n result must be bitwise symmetric (checked
    on the device by the require_symmetric kernel)."""
    import torch
    from paper_2410_19208_b200 import workloads
    from paper_2410_19208_b200.symmetric import check_symmetric_device
    from paper_2410_19208_b200._tensors import Operand
    n, k, p, q = 32768, 256, 16, 1
    dev = torch.device("cuda", 0)
    xd = workloads.c3_device(n, seed=seed, device=dev)
    om = np.random.default_rng(seed + 100).standard_normal((n, k + p))
    rep = ours.ran_proj(xd, ours.RangeParams(k=k, l=p, q=q), None, omega=torch.from_numpy(om).to(dev))
    assert rep.device_info["sketch_engine"] == 1 and rep.device_info["recon_engine"] == 1
    stats = check_symmetric_device(Operand(rep.result, "torch_cuda", dev))
    assert stats.bitwise and stats.defect == 0.0
    res = rep.result.cpu().numpy()
    x = xd.cpu().numpy()
    del xd, rep
    torch.cuda.empty_cache()
    o = orc.ran_proj(x, k, p, q, omega=om)
    del x
    assert res.shape == o.result.shape
    err = _rel(res, o.result)
    assert err <= TOL, err


def test_config4_shape_reduced_n(ours):
    """C4's k = 512, p = 32, q = 2 (w = 544: the INT8 engine runs the panel as two
    column groups; q = 2 re-orthonormalises between products) at n = 8192, through
    the row-sharded driver with the real kernels on one rank, X from the C4 row
    generator (bitwise symmetric, checked)."""
    import torch
    from paper_2410_19208_b200 import workloads
    from paper_2410_19208_b200.sharded import KernelOps, sharded_ran_proj
    n, k, p, q = 8192, 512, 32, 2
    xd = workloads.c4_rows(n, 0, n, seed=5)
    om = np.random.default_rng(6).standard_normal((n, k + p))
    ops = KernelOps("cuda")
    rep = sharded_ran_proj(xd, 0, n, torch.from_numpy(om).cuda(), ours.RangeParams(k=k, l=p, q=q),
                           ops=ops)
    assert ops.int8_products == 2 * q + 2 and rep.bitwise_symmetric is True
    res = rep.result_rows.cpu().numpy()
    ref = orc.ran_proj(xd.cpu().numpy(), k, p, q, omega=om)
    assert rep.basis_width == ref.basis_width and rep.effective_rank == ref.effective_rank
    assert np.array_equal(res, res.T)
    err = _rel(res, ref.result)
    if err > TOL:   # locate the damage (128×128 tiles) before failing
        d = np.abs(res - ref.result).reshape(n // 128, 128, n // 128, 128).max(axis=(1, 3))
        bad = np.argwhere(d > 1e-9 * np.abs(ref.result).max())
        print(f"config4 shape: rel err {err:.3e}; {len(bad)} of {d.size} tiles off, first {bad[:8].tolist()}; "
              f"factor d err {float(np.abs(np.sort(rep.factors_d.cpu().numpy()) - np.sort(ref.factors[1])).max()):.3e}")
    assert err <= TOL


@pytest.mark.parametrize("alpha", [0.0, 0.5])
def test_sharded_single_rank_transposed_branch(ours, alpha):
    """X symmetric only within tolerance: the sharded driver's Xᵀ product takes the
    reduce-scatter branch (Σ_h X_hᵀ Y_h on the DMMA A-transposed kernel; one rank
    here) and must reproduce the reference's x.T @ y (sketch.py:79)."""
    import torch
    from paper_2410_19208_b200.sharded import KernelOps, sharded_ran_proj
    n, k, l, q = 1500, 40, 8, 2
    x = orc.wigner(n, seed=31) + 3e-12 * np.random.default_rng(32).standard_normal((n, n))
    om = np.random.default_rng(33).standard_normal((n, k + l))
    ref = orc.ran_proj_scal(x, k, l, q, alpha, omega=om) if alpha > 0 else orc.ran_proj(x, k, l, q, omega=om)
    rep = sharded_ran_proj(torch.from_numpy(x).cuda(), 0, n, torch.from_numpy(om).cuda(),
                           ours.RangeParams(k=k, l=l, q=q), alpha=alpha, ops=KernelOps("cuda"))
    assert rep.bitwise_symmetric is False
    assert rep.effective_rank == ref.effective_rank
    assert _rel(rep.result_rows.cpu().numpy(), ref.result) <= TOL
    bad = x.copy()
    bad[3, 1000] += 1e-6
    with pytest.raises(ours.AsymmetricMatrixError):
        sharded_ran_proj(torch.from_numpy(bad).cuda(), 0, n, torch.from_numpy(om).cuda(),
                         ours.RangeParams(k=k, l=l, q=q), ops=KernelOps("cuda"))


def test_solver_config5_shape_trajectory(ours):
    """A config-5-shaped run (sparse A_i with 4 mirrored off-diagonal N(0,1) entries,
    C = Wigner + 2I, β = 1/L, randomized projector k = 64, q = 1) at n = 1024,
    m = 4000 for 50 iterations against the oracle's sparse restatement of
    psdcone.solve (sdls.py:164-265) on the same numpy stream."""
    from oracle import sdls_oracle as so
    n, m, k, p, q, its = 1024, 4000, 64, 10, 1, 50
    sp = so.config5_instance(n, m, nnz_per=4, seed=55)
    beta = so.lipschitz_beta(sp)
    ref = so.solve(sp, "randomized", k, p, q, beta=beta, epsilon=1e-300, max_iter=its, rng=9,
                   exact_check_dim=0)
    prob = ours.SparseSdlsProblem(sp.c, 1.0, sp.con, sp.rows, sp.cols, sp.vals, sp.b)
    cfg = ours.ProjectorConfig(method="randomized", params=ours.RangeParams(k=k, l=p, q=q))
    rep = ours.solve(prob, cfg, beta=beta, epsilon=1e-300, max_iter=its, rng=9, keep_trajectory=True,
                     exact_check_dim=0)
    assert rep.iterations == ref.iterations == its
    np.testing.assert_allclose([t.grad_norm for t in rep.trajectory], ref.trajectory, rtol=1e-8)
    np.testing.assert_allclose(rep.y_final, ref.y_final, rtol=1e-8, atol=1e-10)
    assert _rel(rep.x_solution, ref.x_solution) <= 1e-9


@pytest.mark.parametrize("name", ["sdls_exact", "sdls_polar"])
def test_solver_dense_projectors_match_reference(ours, name):
    """solve() with the exact (reference default) / polar projector vs the reference."""
    d = gio.load(name)
    prob = ours.SparseSdlsProblem(d["c"], 1.0, d["con"], d["rows"], d["cols"], d["vals"], d["b"])
    cfg = None if str(d["method"]) == "exact" else ours.ProjectorConfig(method="polar")
    rep = ours.solve(prob, cfg, beta=float(d["beta"]), epsilon=1e-14, max_iter=20, rng=int(d["seed"]),
                     keep_trajectory=True)
    assert rep.iterations == int(d["iterations"])
    np.testing.assert_allclose([t.grad_norm for t in rep.trajectory], d["grad_norms"], rtol=1e-8)
    np.testing.assert_allclose(rep.y_final, d["y_final"], rtol=1e-8, atol=1e-11)
    assert _rel(rep.x_solution, d["x_solution"]) <= 1e-9
    assert rep.objective == pytest.approx(float(d["objective"]), rel=1e-8)
