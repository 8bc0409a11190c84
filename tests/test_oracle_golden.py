"""The CPU oracle (oracle/psd_oracle.py) against the reference's own outputs.

These fixtures were produced by tests/golden/make_golden.py, which runs the
unmodified reference package.  Passing here is what pins the oracle."""

import numpy as np
import pytest

from oracle import psd_oracle as orc
from tests import golden_io as gio

RAN_CASES = [n for n in gio.names() if "w" in np.load(f"{gio.GOLDEN}/{n}.npz").files
             and not n.startswith(("project_", "config1_project"))]


@pytest.mark.parametrize("name", RAN_CASES)
def test_ran_proj_matches_reference(name):
    d = gio.load(name)
    k, l, q = int(d["k"]), int(d["l"]), int(d["q"])
    alpha = float(d["alpha"])
    if alpha > 0:
        rep = orc.ran_proj_scal(d["x"], k, l, q, alpha, omega=d["omega"])
    else:
        rep = orc.ran_proj(d["x"], k, l, q, omega=d["omega"], collect_diagnostics=True)
    ref = gio.golden_result(d)
    assert rep.effective_rank == int(d["effective_rank"])
    assert rep.basis_width == int(d["basis_width"])
    err = np.linalg.norm(rep.result - ref) / max(np.linalg.norm(ref), 1e-300)
    assert err <= 1e-13 or np.linalg.norm(ref) == 0.0, err
    if "result" in d:
        # same numpy calls in the same order: bit-exact in this container
        np.testing.assert_array_equal(rep.result, d["result"])


@pytest.mark.parametrize("name", gio.names("project_") + ["config1_project_scaled"])
def test_project_scaled_matches_reference(name):
    d = gio.load(name)
    k, l, q = int(d["k"]), int(d["l"]), int(d["q"])
    if "alpha_override" in d:
        rep = orc.project_scaled(d["x"], k, l, q, alpha_override=float(d["alpha_override"]),
                                 omega=d["omega"])
    else:
        rep = orc.project_scaled(d["x"], k, l, q, power_n=int(d["power_n"]),
                                 scale_factor=float(d["scale_factor"]),
                                 v1=d["v1"], v2=d["v2"], omega=d["omega"])
    assert rep.fallback == bool(d["fallback"])
    assert rep.alpha_used == pytest.approx(float(d["alpha_used"]), rel=1e-14)
    assert rep.effective_rank == int(d["effective_rank"])
    ref = gio.golden_result(d)
    err = np.linalg.norm(rep.result - ref) / max(np.linalg.norm(ref), 1e-300)
    assert err <= 1e-13, err


@pytest.mark.parametrize("name", gio.names("power_iteration_"))
def test_power_iteration_matches_reference(name):
    d = gio.load(name)
    val = orc.power_iteration(d["x"], int(d["n_iter"]), v0=d["v0"])
    assert val == float(d["value"])


@pytest.mark.parametrize("name", gio.names("min_eig_"))
def test_min_eig_matches_reference(name):
    d = gio.load(name)
    val = orc.min_eig_magnitude(d["x"], int(d["n_iter"]), v1=d["v1"], v2=d["v2"])
    assert val == float(d["value"])


def test_eigh_convention_matches_reference():
    d = gio.load("eigh_wigner50")
    dec = orc.eigh(d["x"])
    np.testing.assert_array_equal(dec.values, d["values"])
    np.testing.assert_array_equal(dec.vectors, d["vectors"])


def test_spec_known_answers():
    # Counterexample 1 at full width, and the scaled fix at k=1.
    d = gio.load("spec_counterexample_full")
    np.testing.assert_allclose(d["result"], np.diag([0.0, 0.0, 1.0]), atol=1e-9)
    d = gio.load("spec_scal_alpha3_k1")   # "≈ diag([0,0,1])" after one power step
    assert d["result"][2, 2] > 0.95 and abs(d["result"][0, 0]) < 1e-12
    assert float(gio.load("min_eig_diag_m3m21")["value"]) == pytest.approx(3.0, rel=1e-2)
    assert float(gio.load("min_eig_diag_123")["value"]) == pytest.approx(1.0, rel=1e-5)
    assert float(gio.load("power_iteration_diag51")["value"]) == pytest.approx(5.0, rel=1e-5)
    assert float(gio.load("power_iteration_zero")["value"]) == 0.0
    assert int(gio.load("rank1_truncation")["basis_width"]) == 1
    assert int(gio.load("zero_matrix")["basis_width"]) == 0


def test_oracle_errors():
    with pytest.raises(orc.OracleError) as e:
        orc.require_symmetric(np.array([[1.0, 2.0], [0.0, 1.0]]))
    assert e.value.kind == "AsymmetricMatrixError"
    with pytest.raises(orc.OracleError) as e:
        orc.ran_proj(np.eye(3), 3, 1, 0, omega=np.ones((3, 4)))
    assert e.value.kind == "InvalidParams"
    with pytest.raises(orc.OracleError) as e:
        orc.ran_proj_scal(np.eye(3), 1, 1, 0, 1e-13, omega=np.ones((3, 2)))
    assert e.value.kind == "AlphaTooSmall"
