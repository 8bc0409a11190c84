"""The drop-in boundary exercised through the REFERENCE's own objects.

``install(psdcone)`` rebinds the reference package onto this path (SURVEY
§8(b)); these tests then call ``psdcone.project`` / ``ran_proj`` /
``range_finder`` / ``solve`` / ``experiments.projection_error_sweep`` with
psdcone's own ``ProjectorConfig`` (projection.py:24-49 — it has no ``dtype``
field), ``RangeParams`` (sketch.py:15-39) and ``SdlsProblem`` (sdls.py:21-57),
and compare against fixtures produced by the un-installed reference
(tests/golden/*.npz) or, where noted, against the reference computed in the
same process before ``install()``.

The reference comes from ``oracle/_ref`` (offline pip install made by
``oracle/make_ref.sh``; it ships to the GPU box) or ``/root/reference``.
"""

import numpy as np
import pytest

from oracle import refpkg
from tests import golden_io as gio

psdcone = refpkg.import_psdcone()
pytestmark = pytest.mark.skipif(psdcone is None, reason="reference package psdcone not installed "
                                                       "(run oracle/make_ref.sh)")


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


@pytest.fixture
def installed():
    import paper_2410_19208_b200 as ours
    ours.install(psdcone)
    try:
        yield ours
    finally:
        ours.uninstall()


def test_install_survives_reference_configs_without_gpu(installed):
    """CPU-side guard for the round-1 crash: a reference ProjectorConfig reaching the
    rebound ``project`` must get as far as the device check (DeviceError without a
    GPU, a report with one) — never AttributeError on a field psdcone lacks."""
    import torch
    cfg = psdcone.ProjectorConfig(method="randomized", params=psdcone.RangeParams(k=2, l=1, q=0))
    x = np.diag([3.0, -1.0, 2.0, 0.5])
    if torch.cuda.is_available():
        rep = psdcone.project(x, cfg, 0)
        assert rep.method == "randomized"
    else:
        with pytest.raises(psdcone.PsdconeError):
            psdcone.project(x, cfg, 0)
    assert installed.errors.REGISTRY["DeviceError"] is not None


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["wigner64_q0", "wigner64_q1", "wigner64_q2", "wigner64_q3",
                                  "c3like_n512_q1", "rank1_truncation", "nearsym96_q1"])
def test_reference_project_randomized(installed, name):
    """psdcone.project(x, psdcone.ProjectorConfig('randomized', ...), seed) — the
    SURVEY §3(A) call stack — through the rebound dispatcher."""
    d = gio.load(name)
    params = psdcone.RangeParams(k=int(d["k"]), l=int(d["l"]), q=int(d["q"]))
    cfg = psdcone.ProjectorConfig(method="randomized", params=params, return_factors=True,
                                  collect_diagnostics=True)
    rep = psdcone.project(d["x"], cfg, int(d["seed"]))
    assert rep.method == "randomized"
    assert _rel(rep.result, gio.golden_result(d)) <= 1e-10
    assert rep.effective_rank == int(d["effective_rank"])
    assert rep.basis_width == int(d["basis_width"])
    w, dd = rep.factors
    np.testing.assert_allclose(np.sort(dd), np.sort(d["d"]), rtol=1e-9, atol=1e-12)
    if "residual_frob" in d:
        assert rep.residual_frob == pytest.approx(float(d["residual_frob"]), rel=1e-7, abs=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["project_scaled_est_wigner80", "project_scaled_half_wigner80",
                                  "config1_project_scaled"])
def test_reference_project_scaled_estimated_alpha(installed, name):
    """Scaled method with α estimated inside project (v1, v2, Ω draw order)."""
    d = gio.load(name)
    params = psdcone.RangeParams(k=int(d["k"]), l=int(d["l"]), q=int(d["q"]))
    cfg = psdcone.ProjectorConfig(method="scaled_randomized", params=params,
                                  power_N=int(d["power_n"]), scale_factor=float(d["scale_factor"]),
                                  return_factors=True)
    rep = psdcone.project(d["x"], cfg, int(d["seed"]))
    assert rep.alpha_used == pytest.approx(float(d["alpha_used"]), rel=1e-10)
    assert bool(rep.fallback) == bool(d["fallback"])
    assert _rel(rep.result, gio.golden_result(d)) <= 1e-10
    assert rep.effective_rank == int(d["effective_rank"])


@pytest.mark.gpu
def test_reference_project_alpha_fallback(installed):
    d = gio.load("project_alpha_fallback")
    cfg = psdcone.ProjectorConfig(method="scaled_randomized",
                                  params=psdcone.RangeParams(k=5, l=2, q=1),
                                  alpha_override=float(d["alpha_override"]), return_factors=True)
    rep = psdcone.project(d["x"], cfg, int(d["seed"]))
    assert rep.fallback is True
    assert rep.alpha_used == pytest.approx(float(d["alpha_used"]))
    assert _rel(rep.result, d["result"]) <= 1e-10


@pytest.mark.gpu
def test_reference_ran_proj_and_ran_proj_scal(installed):
    d = gio.load("wigner64_q2")
    params = psdcone.RangeParams(k=int(d["k"]), l=int(d["l"]), q=int(d["q"]))
    rep = psdcone.ran_proj(d["x"], params, np.random.default_rng(int(d["seed"])),
                           return_factors=True)
    assert _rel(rep.result, d["result"]) <= 1e-10
    s = gio.load("wigner128_scal")
    sp = psdcone.RangeParams(k=int(s["k"]), l=int(s["l"]), q=int(s["q"]))
    rs = psdcone.ran_proj_scal(s["x"], sp, float(s["alpha"]), np.random.default_rng(int(s["seed"])))
    assert rs.method == "scaled_randomized" and rs.alpha_used == pytest.approx(float(s["alpha"]))
    assert _rel(rs.result, s["result"]) <= 1e-10
    with pytest.raises(psdcone.AlphaTooSmall):     # the reference's own exception class
        psdcone.ran_proj_scal(s["x"], sp, 1e-300, np.random.default_rng(0))
    with pytest.raises(psdcone.AsymmetricMatrixError):
        bad = s["x"].copy()
        bad[0, 1] += 1e-3
        psdcone.ran_proj(bad, sp, np.random.default_rng(0))


@pytest.mark.gpu
def test_reference_range_finder_power_and_min_eig(installed):
    """range_finder / power_iteration / min_eig_magnitude under the reference names.
    The basis is compared as the projector QQᵀ (Householder vs CholeskyQR columns
    agree up to sign)."""
    import importlib
    inst = importlib.import_module("paper_2410_19208_b200.install")
    ref_rf = inst.original("psdcone.sketch", "range_finder")
    x = gio.load("wigner64_q1")["x"]
    for q in (0, 1, 2):
        params = psdcone.RangeParams(k=8, l=4, q=q)
        qo = psdcone.range_finder(x, params, np.random.default_rng(5 + q))
        qr = ref_rf(x, params, np.random.default_rng(5 + q))
        assert qo.shape == qr.shape
        assert _rel(qo @ qo.T, qr @ qr.T) <= 1e-10
    p = gio.load("power_iteration_diag51")
    assert psdcone.power_iteration(p["x"], int(p["n_iter"]), np.random.default_rng(1)) == \
        pytest.approx(float(p["value"]), rel=1e-12)
    m = gio.load("min_eig_diag_m3m21")
    assert psdcone.min_eig_magnitude(m["x"], 10, np.random.default_rng(1)) == \
        pytest.approx(float(m["value"]), rel=1e-10)


def _ref_problem(d):
    n, m = int(d["n"]), int(d["m"])
    dense = np.zeros((m, n, n))
    np.add.at(dense, (d["con"], d["rows"], d["cols"]), d["vals"])
    return psdcone.SdlsProblem(d["c"], 1.0, list(zip(dense, d["b"])))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sdls_randomized", "sdls_scaled"])
def test_reference_solve_randomized(installed, name):
    d = gio.load(name)
    cfg = psdcone.ProjectorConfig(method=str(d["method"]),
                                  params=psdcone.RangeParams(k=int(d["k"]), l=int(d["l"]),
                                                             q=int(d["q"])), power_N=10)
    rep = psdcone.solve(_ref_problem(d), cfg, beta=float(d["beta"]), epsilon=1e-14, max_iter=25,
                        rng=int(d["seed"]), alpha_refresh=int(d["alpha_refresh"]),
                        keep_trajectory=True)
    assert rep.iterations == int(d["iterations"])
    np.testing.assert_allclose([t.grad_norm for t in rep.trajectory], d["grad_norms"], rtol=1e-8)
    np.testing.assert_allclose(rep.y_final, d["y_final"], rtol=1e-8, atol=1e-11)
    assert _rel(rep.x_solution, d["x_solution"]) <= 1e-9
    assert rep.exact_feasibility_residual == pytest.approx(float(d["exact_residual"]), rel=1e-7)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sdls_exact", "sdls_polar"])
def test_reference_solve_dense_projectors(installed, name):
    """psdcone.solve(problem) with its default exact projector, and with polar."""
    d = gio.load(name)
    cfg = None if str(d["method"]) == "exact" else psdcone.ProjectorConfig(method="polar")
    rep = psdcone.solve(_ref_problem(d), cfg, beta=float(d["beta"]), epsilon=1e-14, max_iter=20,
                        rng=int(d["seed"]), keep_trajectory=True)
    assert rep.projection_method == str(d["method"])
    assert rep.iterations == int(d["iterations"])
    np.testing.assert_allclose([t.grad_norm for t in rep.trajectory], d["grad_norms"], rtol=1e-8)
    np.testing.assert_allclose(rep.y_final, d["y_final"], rtol=1e-8, atol=1e-11)
    assert _rel(rep.x_solution, d["x_solution"]) <= 1e-9
    assert rep.objective == pytest.approx(float(d["objective"]), rel=1e-8)
    assert rep.exact_feasibility_residual is None


@pytest.mark.gpu
def test_reference_dual_gradient_uses_rebound_project():
    """sdls.dual_gradient is NOT rebound: it calls the rebound ``project`` with a
    reference config.  Compare to the same call before install()."""
    import paper_2410_19208_b200 as ours
    d = gio.load("sdls_randomized")
    prob = _ref_problem(d)
    y = np.random.default_rng(3).standard_normal(int(d["m"]))
    cfg = psdcone.ProjectorConfig(method="randomized", params=psdcone.RangeParams(k=8, l=4, q=1))
    want = psdcone.sdls.dual_gradient(prob, y, cfg, np.random.default_rng(9))
    want_exact = psdcone.sdls.dual_gradient(prob, y)
    ours.install(psdcone)
    try:
        got = psdcone.sdls.dual_gradient(prob, y, cfg, np.random.default_rng(9))
        got_exact = psdcone.sdls.dual_gradient(prob, y)
    finally:
        ours.uninstall()
    assert _rel(got, want) <= 1e-9
    assert _rel(got_exact, want_exact) <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sweep_fourblock_q0", "sweep_fourblock_q1"])
def test_reference_projection_error_sweep(installed, name):
    d = gio.load(name)
    rows = psdcone.experiments.projection_error_sweep(
        int(d["n"]), psdcone.experiments.FOUR_BLOCK_BETAS, int(d["l"]), int(d["q"]),
        [int(k) for k in d["k_grid"]], int(d["trials"]), int(d["seed"]))
    assert len(rows) == len(d["k"])
    for i, r in enumerate(rows):
        assert r.k == int(d["k"][i])
        assert r.mean_frob_error == pytest.approx(float(d["mean_frob"][i]), rel=1e-6, abs=1e-8)
        assert r.mean_spectral_error == pytest.approx(float(d["mean_spec"][i]), rel=1e-6, abs=1e-8)
