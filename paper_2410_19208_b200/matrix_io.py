"""File formats on either side of the projection path (SPEC.md
`matrix_io`): Matrix Market matrices and JSON SDLS problem files.

The reference declares these formats (`pkg/pyproject.toml:16`)
but ships no implementation, so this module restates the published Matrix
Market rules:

* header ``%%MatrixMarket matrix <format> <field> <symmetry>`` with format
  ``coordinate`` | ``array``, field ``real`` | ``double`` | ``integer`` |
  ``pattern`` (coordinate only), symmetry ``general`` | ``symmetric`` |
  ``skew-symmetric``; ``%`` comment lines; then the size line;
* coordinate: 1-based ``i j [value]`` triplets; for symmetric /
  skew-symmetric files only entries with i ≥ j are stored and the reader
  mirrors them (duplicate entries are summed, as common readers do);
* array: values in column-major order; symmetric / skew-symmetric arrays
  store the lower triangle column by column.

Values are written with 17 significant digits, so ``read(write(X))``
reproduces X bit for bit.  Parse errors raise ``InvalidParams`` carrying
``path:line:column``.  ``device=`` hands the matrix straight to HBM as a
float64 CUDA tensor ready for ``ran_proj`` / ``project``.
"""

from __future__ import annotations

import io
import json
import os

import numpy as np

from . import errors

_FORMATS = ("coordinate", "array")
_FIELDS = ("real", "double", "integer", "pattern")
_SYMM = ("general", "symmetric", "skew-symmetric")


def _err(src, line, col, msg):
    return errors.error("InvalidParams", f"{src}:{line}:{col}: {msg}")


def _open_text(path_or_file, mode):
    if isinstance(path_or_file, (str, os.PathLike)):
        return open(path_or_file, mode, encoding="ascii"), str(path_or_file), True
    return path_or_file, getattr(path_or_file, "name", "<stream>"), False


def _number(tok, src, line, col, integer):
    try:
        return float(int(tok)) if integer else float(tok)
    except ValueError:
        raise _err(src, line, col, f"expected {'an integer' if integer else 'a real'} value, got {tok!r}")


def read_matrix_market(path_or_file, *, device=None):
    """Read a Matrix Market file into a dense float64 matrix (numpy, or a CUDA
    tensor on ``device``)."""
    fh, src, close = _open_text(path_or_file, "r")
    try:
        lines = fh.read().splitlines()
    finally:
        if close:
            fh.close()
    if not lines:
        raise _err(src, 1, 1, "empty file")
    head = lines[0].split()
    if len(head) != 5 or head[0] != "%%MatrixMarket" or head[1].lower() != "matrix":
        raise _err(src, 1, 1, "expected header '%%MatrixMarket matrix <format> <field> <symmetry>'")
    fmt, field, symm = (h.lower() for h in head[2:])
    for val, allowed, pos in ((fmt, _FORMATS, 3), (field, _FIELDS, 4), (symm, _SYMM, 5)):
        if val not in allowed:
            col = len(" ".join(head[:pos - 1])) + 2
            raise _err(src, 1, col, f"unsupported {('format', 'field', 'symmetry')[pos - 3]} {val!r}")
    if field == "pattern" and fmt == "array":
        raise _err(src, 1, 1, "pattern field is only valid for coordinate matrices")
    # data tokens with their (line, column) for error reporting
    li = 1
    while li < len(lines) and (not lines[li].strip() or lines[li].lstrip().startswith("%")):
        li += 1
    if li >= len(lines):
        raise _err(src, li + 1, 1, "missing size line")
    size_tok = lines[li].split()
    want = 3 if fmt == "coordinate" else 2
    if len(size_tok) != want:
        raise _err(src, li + 1, 1, f"size line needs {want} integers, got {len(size_tok)}")
    try:
        dims = [int(t) for t in size_tok]
    except ValueError:
        raise _err(src, li + 1, 1, "size line must hold integers")
    nr, nc = dims[0], dims[1]
    if nr < 0 or nc < 0 or (symm != "general" and nr != nc):
        raise _err(src, li + 1, 1, f"invalid dimensions {nr}x{nc} for a {symm} matrix")
    integer = field == "integer"
    body = [(k + 1, ln) for k, ln in enumerate(lines[li + 1:], start=li + 1)
            if ln.strip() and not ln.lstrip().startswith("%")]
    x = np.zeros((nr, nc), dtype=np.float64)
    if fmt == "coordinate":
        nnz = dims[2]
        if len(body) != nnz:
            at = body[min(len(body), nnz) - 1][0] + 1 if body else li + 2
            raise _err(src, at, 1, f"expected {nnz} entries, found {len(body)}")
        per = 2 if field == "pattern" else 3
        ii = np.empty(nnz, dtype=np.int64)
        jj = np.empty(nnz, dtype=np.int64)
        vv = np.ones(nnz, dtype=np.float64)
        for t, (lno, ln) in enumerate(body):
            tok = ln.split()
            if len(tok) != per:
                raise _err(src, lno, 1, f"expected {per} fields, got {len(tok)}")
            try:
                i, j = int(tok[0]), int(tok[1])
            except ValueError:
                raise _err(src, lno, 1, "row/column indices must be integers")
            if not (1 <= i <= nr and 1 <= j <= nc):
                raise _err(src, lno, 1, f"index ({i}, {j}) outside {nr}x{nc}")
            if symm != "general" and i < j:
                raise _err(src, lno, 1, f"{symm} files store only i >= j entries, got ({i}, {j})")
            if symm == "skew-symmetric" and i == j:
                raise _err(src, lno, 1, "skew-symmetric files have no diagonal entries")
            if per == 3:
                vv[t] = _number(tok[2], src, lno, len(tok[0]) + len(tok[1]) + 3, integer)
            ii[t], jj[t] = i - 1, j - 1
        np.add.at(x, (ii, jj), vv)
        if symm != "general":
            off = ii != jj
            sign = -1.0 if symm == "skew-symmetric" else 1.0
            np.add.at(x, (jj[off], ii[off]), sign * vv[off])
    else:
        vals = []
        for lno, ln in body:
            tok = ln.split()
            if len(tok) != 1:
                raise _err(src, lno, 1, f"array files hold one value per line, got {len(tok)}")
            vals.append(_number(tok[0], src, lno, 1, integer))
        if symm == "general":
            need = nr * nc
        elif symm == "symmetric":
            need = nr * (nr + 1) // 2
        else:
            need = nr * (nr - 1) // 2
        if len(vals) != need:
            at = body[-1][0] + 1 if body else li + 2
            raise _err(src, at, 1, f"expected {need} values, found {len(vals)}")
        v = np.asarray(vals, dtype=np.float64)
        if symm == "general":
            x = v.reshape(nc, nr).T.copy()
        else:
            t = 0
            for j in range(nc):                     # lower triangle, column by column
                i0 = j if symm == "symmetric" else j + 1
                cnt = nr - i0
                x[i0:, j] = v[t:t + cnt]
                t += cnt
            lower = np.tril(x, -1)
            x = x + (lower.T if symm == "symmetric" else -lower.T)
    if device is not None:
        import torch
        return torch.from_numpy(x).to(device)
    return x


def write_matrix_market(path_or_file, x, *, fmt="array", symmetry=None, comment=None):
    """Write a dense matrix.  ``fmt``: "array" (column-major values) or
    "coordinate" (nonzeros); ``symmetry``: "general" | "symmetric" |
    "skew-symmetric" | None (symmetric if X is bitwise symmetric, else general).
    17 significant digits: ``read(write(X))`` is exact."""
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2:
        raise errors.error("InvalidParams", f"expected a 2-D matrix, got shape {x.shape}")
    if fmt not in _FORMATS:
        raise errors.error("InvalidParams", f"format must be one of {_FORMATS}, got {fmt!r}")
    nr, nc = x.shape
    if symmetry is None:
        symmetry = "symmetric" if nr == nc and np.array_equal(x, x.T) else "general"
    if symmetry not in _SYMM:
        raise errors.error("InvalidParams", f"symmetry must be one of {_SYMM}, got {symmetry!r}")
    if symmetry != "general":
        if nr != nc:
            raise errors.error("NonSquareError", f"{symmetry} output needs a square matrix, got {x.shape}")
        ref = x.T if symmetry == "symmetric" else -x.T
        if not np.array_equal(x, ref):
            raise errors.error("InvalidParams", f"matrix is not exactly {symmetry}")
    out = io.StringIO()
    out.write(f"%%MatrixMarket matrix {fmt} real {symmetry}\n")
    if comment:
        for ln in str(comment).splitlines():
            out.write(f"% {ln}\n")
    if fmt == "array":
        out.write(f"{nr} {nc}\n")
        for j in range(nc):
            if symmetry == "general":
                col = x[:, j]
            else:
                col = x[(j if symmetry == "symmetric" else j + 1):, j]
            if col.size:
                out.write("\n".join(f"{v:.17g}" for v in col))
                out.write("\n")
    else:
        if symmetry == "general":
            ii, jj = np.nonzero(x)
        else:
            ii, jj = np.nonzero(np.tril(x, 0 if symmetry == "symmetric" else -1))
        order = np.lexsort((ii, jj))                 # column-major entry order
        ii, jj = ii[order], jj[order]
        out.write(f"{nr} {nc} {ii.size}\n")
        for i, j in zip(ii, jj):
            out.write(f"{i + 1} {j + 1} {x[i, j]:.17g}\n")
    fh, _, close = _open_text(path_or_file, "w")
    try:
        fh.write(out.getvalue())
    finally:
        if close:
            fh.close()


# --------------------------------------------------------- SDLS problem files --

def _matrix_from_json(obj, n, where, base_dir):
    """A matrix reference: a Matrix Market path (relative to the problem file),
    inline triplets {"n": n, "triplets": [[i, j, v], ...], "symmetric": bool}
    (0-based), or a dense nested list."""
    if isinstance(obj, str):
        p = obj if os.path.isabs(obj) or base_dir is None else os.path.join(base_dir, obj)
        return read_matrix_market(p)
    if isinstance(obj, dict):
        size = int(obj.get("n", n))
        m = np.zeros((size, size))
        sym = bool(obj.get("symmetric", True))
        for t, trip in enumerate(obj.get("triplets", [])):
            if len(trip) != 3:
                raise errors.error("InvalidParams", f"{where}: triplet {t} must be [i, j, value]")
            i, j, v = int(trip[0]), int(trip[1]), float(trip[2])
            if not (0 <= i < size and 0 <= j < size):
                raise errors.error("InvalidParams", f"{where}: triplet {t} index ({i}, {j}) outside {size}x{size}")
            m[i, j] += v
            if sym and i != j:
                m[j, i] += v
        return m
    if isinstance(obj, list):
        return np.asarray(obj, dtype=float)
    raise errors.error("InvalidParams", f"{where}: unsupported matrix encoding {type(obj).__name__}")


def read_sdls_problem(path_or_file):
    """JSON problem file {n, rho, C, constraints: [{A, b}]} → SparseSdlsProblem
    (constraints kept as COO triplets; C dense)."""
    from .sdls import SparseSdlsProblem
    fh, src, close = _open_text(path_or_file, "r")
    try:
        try:
            d = json.load(fh)
        except json.JSONDecodeError as exc:
            raise _err(src, exc.lineno, exc.colno, exc.msg)
    finally:
        if close:
            fh.close()
    base = os.path.dirname(os.path.abspath(src)) if isinstance(path_or_file, (str, os.PathLike)) else None
    for key in ("n", "rho", "C", "constraints"):
        if key not in d:
            raise errors.error("InvalidParams", f"{src}: missing field {key!r}")
    n = int(d["n"])
    c = _matrix_from_json(d["C"], n, f"{src}: C", base)
    if c.shape != (n, n):
        raise errors.error("DimensionMismatch", f"{src}: C is {c.shape}, expected ({n}, {n})")
    con, rows, cols, vals, b = [], [], [], [], []
    for k, item in enumerate(d["constraints"]):
        if "A" not in item or "b" not in item:
            raise errors.error("InvalidParams", f"{src}: constraint {k} needs fields 'A' and 'b'")
        a = _matrix_from_json(item["A"], n, f"{src}: constraint {k}", base)
        if a.shape != (n, n):
            raise errors.error("DimensionMismatch", f"{src}: constraint {k} A is {a.shape}, expected ({n}, {n})")
        r, cc = np.nonzero(a)
        con.append(np.full(r.size, k))
        rows.append(r)
        cols.append(cc)
        vals.append(a[r, cc])
        b.append(float(item["b"]))
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dtype=dt))
    return SparseSdlsProblem(c, float(d["rho"]), cat(con, np.int64), cat(rows, np.int64),
                             cat(cols, np.int64), cat(vals, float), np.asarray(b, dtype=float))


def write_sdls_problem(path_or_file, problem):
    """SparseSdlsProblem → JSON with inline 0-based triplets (17 significant digits)."""
    c = np.asarray(problem.c, dtype=float)
    n = c.shape[0]
    ci, cj = np.nonzero(c)
    doc = {"n": n, "rho": float(problem.rho),
           "C": {"n": n, "symmetric": False,
                 "triplets": [[int(i), int(j), float(c[i, j])] for i, j in zip(ci, cj)]},
           "constraints": []}
    for k in range(problem.m):
        sel = problem.con == k
        doc["constraints"].append({
            "A": {"n": n, "symmetric": False,
                  "triplets": [[int(i), int(j), float(v)] for i, j, v in
                               zip(problem.rows[sel], problem.cols[sel], problem.vals[sel])]},
            "b": float(problem.b[k])})
    text = json.dumps(doc, indent=1)          # json floats use repr: 17-digit round trip
    fh, _, close = _open_text(path_or_file, "w")
    try:
        fh.write(text)
    finally:
        if close:
            fh.close()


__all__ = ["read_matrix_market", "write_matrix_market", "read_sdls_problem", "write_sdls_problem"]
