"""§8 f3: the Monte-Carlo projection-error harness (experiments.py:78-137) and
its closed-form bounds (bounds.py), against fixtures produced by the real
reference (tests/golden/make_golden.py: sweep_cases)."""

import numpy as np
import pytest

from tests import golden_io as gio


@pytest.fixture(scope="module")
def ex():
    from paper_2410_19208_b200 import experiments
    return experiments


def test_four_block_matrix_matches_reference(ex):
    for name in ("sweep_fourblock_q0", "sweep_fourblock_q1"):
        d = gio.load(name)
        x = ex.four_block_matrix(int(d["n"]), ex.FOUR_BLOCK_BETAS, int(d["seed"]))
        np.testing.assert_array_equal(x, d["x"])


def test_bounds_match_reference(ex):
    d = gio.load("bounds_generic")
    spec = ex.SpectrumSummary.from_eigenvalues(d["eigenvalues"])
    for row in d["table"]:
        k, l, q, alpha = int(row[0]), int(row[1]), int(row[2]), float(row[3])
        p = ex.BoundParams(k=k, l=l, q=q)
        got = [ex.eps1(spec.sigmas, k, l), ex.eps2(spec.sigmas[k], k, l, q, spec.n),
               ex.frob_bound_unscaled(spec, p) if q == 0 else np.nan,
               ex.spectral_bound_unscaled(spec, p),
               ex.frob_bound_scaled(spec, p, alpha) if q == 0 else np.nan,
               ex.spectral_bound_scaled(spec, p, alpha)]
        np.testing.assert_allclose(got, row[4:], rtol=1e-13, equal_nan=True)


def test_bound_validation(ex):
    with pytest.raises(Exception):
        ex.BoundParams(k=2, l=1)
    with pytest.raises(Exception):
        ex.four_block_eigenvalues(10, ex.FOUR_BLOCK_BETAS)
    spec = ex.SpectrumSummary.from_eigenvalues(ex.four_block_eigenvalues(16, ex.FOUR_BLOCK_BETAS))
    with pytest.raises(Exception):
        ex.frob_bound_unscaled(spec, ex.BoundParams(k=4, l=3, q=1))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sweep_fourblock_q0", "sweep_fourblock_q1"])
def test_projection_error_sweep_gpu(ex, name):
    d = gio.load(name)
    rows = ex.projection_error_sweep(int(d["n"]), ex.FOUR_BLOCK_BETAS, int(d["l"]), int(d["q"]),
                                     [int(k) for k in d["k_grid"]], int(d["trials"]), int(d["seed"]))
    methods = {0: "randomized", 1: "scaled_randomized"}
    assert len(rows) == len(d["k"])
    for i, r in enumerate(rows):
        assert r.k == int(d["k"][i]) and r.method == methods[int(d["method"][i])]
        # the projections agree with the reference to ≤1e-10 relative; the errors are
        # differences of O(1) matrices, so compare them to 1e-8 of the matrix scale
        assert r.mean_frob_error == pytest.approx(float(d["mean_frob"][i]), rel=1e-6, abs=1e-8)
        assert r.mean_spectral_error == pytest.approx(float(d["mean_spec"][i]), rel=1e-6, abs=1e-8)
        fb = float(d["frob_bound"][i])
        if np.isnan(fb):
            assert r.frob_bound is None
        else:
            assert r.frob_bound == pytest.approx(fb, rel=1e-13)
        assert r.spectral_bound == pytest.approx(float(d["spec_bound"][i]), rel=1e-13)
