"""§8 f4 data formats: Matrix Market matrices and JSON SDLS problem files
(SPEC.md matrix_io examples: exact round trip of diag([−3,−2,1]), symmetric
coordinate files store i ≥ j and the reader mirrors, malformed headers report
their location)."""

import io

import numpy as np
import pytest

from paper_2410_19208_b200 import errors, matrix_io as mio


def _rt(x, **kw):
    buf = io.StringIO()
    mio.write_matrix_market(buf, x, **kw)
    buf.seek(0)
    return buf.getvalue(), mio.read_matrix_market(io.StringIO(buf.getvalue()))


def test_diag_round_trip_exact():
    x = np.diag([-3.0, -2.0, 1.0])
    for fmt in ("array", "coordinate"):
        text, y = _rt(x, fmt=fmt)
        assert text.startswith(f"%%MatrixMarket matrix {fmt} real symmetric")
        np.testing.assert_array_equal(y, x)


def test_random_round_trip_bitwise_17_digits():
    rng = np.random.default_rng(0)
    g = rng.standard_normal((23, 17)) * 10.0 ** rng.integers(-300, 300, (23, 17))
    for fmt in ("array", "coordinate"):
        _, y = _rt(g, fmt=fmt)
        assert y.tobytes() == g.tobytes()
    s = rng.standard_normal((19, 19))
    s = s + s.T
    for fmt in ("array", "coordinate"):
        text, y = _rt(s, fmt=fmt)
        assert "symmetric" in text.splitlines()[0]
        assert y.tobytes() == s.tobytes()
    k = np.triu(rng.standard_normal((7, 7)), 1)
    k = k - k.T
    for fmt in ("array", "coordinate"):
        _, y = _rt(k, fmt=fmt, symmetry="skew-symmetric")
        np.testing.assert_array_equal(y, k)


def test_coordinate_symmetric_stores_lower_and_mirrors():
    text = ("%%MatrixMarket matrix coordinate real symmetric\n% a comment\n\n"
            "3 3 4\n1 1 2.5\n3 1 -1\n2 2 4\n3 3 1e-3\n")
    x = mio.read_matrix_market(io.StringIO(text))
    np.testing.assert_array_equal(x, [[2.5, 0, -1], [0, 4, 0], [-1, 0, 1e-3]])
    _, y = _rt(x, fmt="coordinate")
    np.testing.assert_array_equal(y, x)
    with pytest.raises(errors.InvalidParams, match=r":4:1: .*only i >= j"):
        mio.read_matrix_market(io.StringIO(
            "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n1 2 3\n"))


def test_pattern_integer_general_and_duplicates():
    x = mio.read_matrix_market(io.StringIO(
        "%%MatrixMarket matrix coordinate pattern general\n2 3 2\n1 3\n2 1\n"))
    np.testing.assert_array_equal(x, [[0, 0, 1], [1, 0, 0]])
    x = mio.read_matrix_market(io.StringIO(
        "%%MatrixMarket matrix coordinate integer general\n2 2 3\n1 1 2\n1 1 3\n2 2 -7\n"))
    np.testing.assert_array_equal(x, [[5, 0], [0, -7]])
    x = mio.read_matrix_market(io.StringIO(
        "%%MatrixMarket matrix array real general\n2 3\n1\n2\n3\n4\n5\n6\n"))
    np.testing.assert_array_equal(x, [[1, 3, 5], [2, 4, 6]])


@pytest.mark.parametrize("text,where", [
    ("%%MatrixMarket matrix banana real general\n1 1\n1\n", ":1:"),
    ("%MatrixMarket matrix array real general\n1 1\n1\n", ":1:1:"),
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n", ":6:1:"),
    ("%%MatrixMarket matrix array real general\n1 1\nx1\n", ":3:1:"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 5 1.0\n", ":3:1:"),
    ("%%MatrixMarket matrix coordinate real general\n2 two 1\n1 1 1.0\n", ":2:1:"),
    ("", ":1:1:"),
])
def test_parse_errors_carry_location(text, where):
    with pytest.raises(errors.InvalidParams, match=where):
        mio.read_matrix_market(io.StringIO(text))


def test_write_validation():
    with pytest.raises(errors.InvalidParams):
        mio.write_matrix_market(io.StringIO(), np.array([[1.0, 2.0], [3.0, 4.0]]), symmetry="symmetric")
    with pytest.raises(errors.InvalidParams):
        mio.write_matrix_market(io.StringIO(), np.eye(2), fmt="csr")


def test_file_paths(tmp_path):
    x = np.arange(9.0).reshape(3, 3)
    p = tmp_path / "m.mtx"
    mio.write_matrix_market(p, x, comment="written by the test")
    np.testing.assert_array_equal(mio.read_matrix_market(p), x)
    assert "% written by the test" in p.read_text()


def test_sdls_problem_round_trip(tmp_path):
    from paper_2410_19208_b200.sdls import SparseSdlsProblem
    c = np.diag([1.0, 2.0, 3.0])
    prob = SparseSdlsProblem(c, 0.5, [0, 0, 1], [0, 1, 2], [1, 0, 2], [0.25, 0.25, -1.5], [1.0, -2.0])
    p = tmp_path / "prob.json"
    mio.write_sdls_problem(p, prob)
    q = mio.read_sdls_problem(p)
    np.testing.assert_array_equal(q.c, c)
    assert q.rho == 0.5 and q.m == 2 and q.n == 3
    np.testing.assert_array_equal(q.b, [1.0, -2.0])
    dense = lambda pr, k: np.bincount(pr.rows[pr.con == k] * 3 + pr.cols[pr.con == k],
                                      pr.vals[pr.con == k], minlength=9).reshape(3, 3)
    for k in range(2):
        np.testing.assert_array_equal(dense(q, k), dense(prob, k))


def test_sdls_problem_matrix_refs_and_errors(tmp_path):
    mio.write_matrix_market(tmp_path / "c.mtx", np.eye(2) * 3)
    (tmp_path / "p.json").write_text('{"n": 2, "rho": 1, "C": "c.mtx", "constraints": '
                                     '[{"A": {"triplets": [[0, 1, 0.5]]}, "b": 1.0}]}')
    q = mio.read_sdls_problem(tmp_path / "p.json")
    np.testing.assert_array_equal(q.c, np.eye(2) * 3)
    assert sorted(zip(q.rows.tolist(), q.cols.tolist())) == [(0, 1), (1, 0)]   # symmetric triplets mirrored
    (tmp_path / "bad.json").write_text('{"n": 2, "rho": 1, "C": [[1, 0], [0, 1]], "constraints": [{"A": [[1, 0], [0, 1]]}]}')
    with pytest.raises(errors.InvalidParams, match="needs fields"):
        mio.read_sdls_problem(tmp_path / "bad.json")
    (tmp_path / "broken.json").write_text('{"n": 2,\n "rho": }')
    with pytest.raises(errors.InvalidParams, match=r"broken.json:2:"):
        mio.read_sdls_problem(tmp_path / "broken.json")


@pytest.mark.gpu
def test_counterexample1_file_to_projection(tmp_path):
    """SPEC matrix_io/cli_project example: diag([−3,−2,1]) from an .mtx file,
    exact projection → diag([0,0,1]); the file loads straight into HBM."""
    import paper_2410_19208_b200 as psd
    p = tmp_path / "ce1.mtx"
    mio.write_matrix_market(p, np.diag([-3.0, -2.0, 1.0]), fmt="coordinate")
    x = mio.read_matrix_market(p, device="cuda")
    assert x.is_cuda and x.dtype.__str__() == "torch.float64"
    rep = psd.project(x, psd.ProjectorConfig(method="exact"))
    np.testing.assert_allclose(rep.result.cpu().numpy(), np.diag([0.0, 0.0, 1.0]), atol=1e-12)
    out = tmp_path / "out.mtx"
    mio.write_matrix_market(out, rep.result)
    np.testing.assert_allclose(mio.read_matrix_market(out), np.diag([0.0, 0.0, 1.0]), atol=1e-12)
