"""Command-line front end (SPEC.md:609-685 harness_cli): exit codes, JSON error
channel, and — on the GPU — the project / solve / fig4 commands end to end."""

import json
import os

import numpy as np
import pytest

from paper_2410_19208_b200 import cli, matrix_io


def _run(capsys, argv):
    code = cli.main(argv)
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def _err(err):
    doc = json.loads(err.strip().splitlines()[-1])
    assert set(doc) == {"error", "message"}
    return doc


def test_bad_flags_exit_2(capsys):
    code, _, err = _run(capsys, ["project", "--input", "x.mtx"])          # missing --output/--method
    assert code == 2 and _err(err)["error"] == "InvalidParams"
    code, _, err = _run(capsys, ["nonsense"])
    assert code == 2


def test_missing_input_exit_2(capsys, tmp_path):
    code, _, err = _run(capsys, ["project", "--input", str(tmp_path / "nope.mtx"), "--output",
                                 str(tmp_path / "o.mtx"), "--method", "exact"])
    assert code == 2 and _err(err)["error"] in ("FileNotFoundError", "InvalidParams")


def test_malformed_header_exit_2_with_location(capsys, tmp_path):
    p = tmp_path / "bad.mtx"
    p.write_text("%%MatrixMarket matrix array\n2 2\n1\n2\n3\n4\n")
    code, _, err = _run(capsys, ["project", "--input", str(p), "--output", str(tmp_path / "o.mtx"),
                                 "--method", "exact"])
    doc = _err(err)
    assert code == 2 and "1" in doc["message"]          # line 1 named in the parse error


def test_k_exceeds_dimension_exit_2(capsys, tmp_path):
    p = tmp_path / "x.mtx"
    matrix_io.write_matrix_market(str(p), np.eye(5))
    code, _, err = _run(capsys, ["project", "--input", str(p), "--output", str(tmp_path / "o.mtx"),
                                 "--method", "randomized", "--k", "10"])
    doc = _err(err)
    assert code == 2 and "k+l exceeds dimension" in doc["message"]
    assert not os.path.exists(tmp_path / "o.mtx")


def test_solve_rejects_exact_and_bad_problem(capsys, tmp_path):
    p = tmp_path / "p.json"
    p.write_text(json.dumps({"n": 2, "rho": 1.0, "C": {"n": 2, "triplets": []},
                             "constraints": [{"A": {"n": 2, "triplets": [[0, 0, 1.0], [1, 1, 1.0]]}}]}))
    code, _, err = _run(capsys, ["solve", "--problem", str(p), "--proj", "randomized", "--k", "1", "--l", "1"])
    assert code == 2 and "'b'" in _err(err)["message"]          # missing b field
    p.write_text(json.dumps({"n": 2, "rho": 1.0, "C": {"n": 2, "triplets": []},
                             "constraints": [{"A": {"n": 2, "triplets": [[0, 0, 1.0], [1, 1, 1.0]]},
                                              "b": 1.0}]}))
    code, _, err = _run(capsys, ["solve", "--problem", str(p), "--proj", "exact"])
    assert code == 2


def test_fig4_beta_order_exit_2(capsys, tmp_path):
    code, _, err = _run(capsys, ["fig4", "--betas", "1,2,3,4", "--out", str(tmp_path / "f.csv")])
    assert code == 2 and "beta3 > beta1" in _err(err)["message"]


@pytest.mark.gpu
def test_project_counterexample_exact(capsys, tmp_path):
    p, o, r = tmp_path / "x.mtx", tmp_path / "o.mtx", tmp_path / "r.json"
    matrix_io.write_matrix_market(str(p), np.diag([-3.0, -2.0, 1.0]))
    code, _, err = _run(capsys, ["project", "--input", str(p), "--output", str(o), "--method", "exact",
                                 "--report", str(r)])
    assert code == 0, err
    np.testing.assert_allclose(matrix_io.read_matrix_market(str(o)), np.diag([0.0, 0.0, 1.0]), atol=1e-12)
    assert json.loads(r.read_text())["effective_rank"] == 1


@pytest.mark.gpu
def test_project_randomized_deterministic(capsys, tmp_path):
    from oracle import psd_oracle as orc
    x = orc.wigner(120, seed=3)
    p = tmp_path / "x.mtx"
    matrix_io.write_matrix_market(str(p), x)
    outs = []
    for t in range(2):
        o, r = tmp_path / f"o{t}.mtx", tmp_path / f"r{t}.json"
        code, _, err = _run(capsys, ["project", "--input", str(p), "--output", str(o), "--method",
                                     "randomized", "--k", "12", "--l", "4", "--q", "1", "--seed", "7",
                                     "--report", str(r)])
        assert code == 0, err
        outs.append((o.read_bytes(), json.loads(r.read_text())))
    assert outs[0][0] == outs[1][0]
    assert {k: v for k, v in outs[0][1].items() if k != "output"} == \
        {k: v for k, v in outs[1][1].items() if k != "output"}
    ref = orc.ran_proj(x, 12, 4, 1, rng=np.random.default_rng(7)).result
    got = matrix_io.read_matrix_market(str(tmp_path / "o0.mtx"))
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-10


@pytest.mark.gpu
def test_solve_tiny_problem(capsys, tmp_path):
    # C = 0, ρ = 1, A₁ = I₂, b = [1]: dual optimum y = 0.5
    p, r = tmp_path / "p.json", tmp_path / "s.json"
    p.write_text(json.dumps({"n": 2, "rho": 1.0, "C": {"n": 2, "triplets": []},
                             "constraints": [{"A": {"n": 2, "triplets": [[0, 0, 1.0], [1, 1, 1.0]]},
                                              "b": 1.0}]}))
    code, _, err = _run(capsys, ["solve", "--problem", str(p), "--proj", "randomized", "--k", "1", "--l", "1",
                                 "--beta", "0.25", "--epsilon", "1e-10", "--max-iter", "200", "--seed", "3",
                                 "--report", str(r)])
    assert code == 0, err
    doc = json.loads(r.read_text())
    assert abs(doc["y_final"][0] - 0.5) <= 1e-8 and doc["feasibility_residual"] <= 1e-8


@pytest.mark.gpu
def test_fig4_csv(capsys, tmp_path):
    out = tmp_path / "f.csv"
    code, _, err = _run(capsys, ["fig4", "--n", "200", "--betas", "3,1,6,2", "--l", "5", "--q", "0",
                                 "--k-grid", "20,40", "--trials", "1", "--seed", "1", "--out", str(out)])
    assert code == 0, err
    lines = out.read_text().splitlines()
    assert lines[0].startswith("k,method,mean_frob_error") and len(lines) == 5
    methods = set()
    for row in lines[1:]:
        k, method, fe, se, fb, sb = row.split(",")
        methods.add(method)
        assert all(np.isfinite(float(v)) and float(v) >= 0 for v in (fe, se, fb, sb))
    assert methods == {"randomized", "scaled_randomized"}
