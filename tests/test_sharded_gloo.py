"""Multi-rank host logic of the row-sharded projection on CPU:
world_size 2 with gloo, numpy stand-in ops, compared with the single-process
oracle on identical X and Ω."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import psd_oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _matrix(n, kind):
    if kind == "rank1":
        u = np.random.default_rng(5).standard_normal(n)
        return np.outer(u, u)
    if kind == "nearsym":   # symmetric only within tolerance: Xᵀ products by reduce-scatter
        x = orc.wigner(n, seed=3)
        return x + 2e-12 * np.random.default_rng(8).standard_normal((n, n))
    if kind == "asym":      # outside the tolerance: AsymmetricMatrixError on every rank
        x = orc.wigner(n, seed=3)
        x[5, n - 3] += 1e-6
        return x
    return orc.wigner(n, seed=3) if kind == "wigner" else orc.c3_matrix(n, seed=4, rank=20)


def _worker(rank, world, port, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2410_19208_b200 import RangeParams
        from paper_2410_19208_b200.sharded import Comm, row_split, sharded_ran_proj
        from tests.numpy_ops import NumpyOps
        n, k, l, q, alpha, kind = case[:6]
        symmetric = case[6] if len(case) > 6 else "check"
        x = _matrix(n, kind)
        om = np.random.default_rng(7).standard_normal((n, k + l))
        starts = row_split(n, world)
        r0, r1 = starts[rank], starts[rank + 1]
        try:
            rep = sharded_ran_proj(torch.from_numpy(x[r0:r1].copy()), r0, n, torch.from_numpy(om),
                                   RangeParams(k=k, l=l, q=q), alpha=alpha, comm=Comm(), ops=NumpyOps(),
                                   symmetric=symmetric)
        except Exception as exc:  # reported to the parent (e.g. AsymmetricMatrixError)
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), error=type(exc).__name__)
            return
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), rows=rep.result_rows.numpy(), r0=r0, r1=r1,
                 eff=rep.effective_rank, width=rep.basis_width,
                 bitwise=-1 if rep.bitwise_symmetric is None else int(rep.bitwise_symmetric))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (96, 10, 6, 1, 0.0, "wigner"),     # unstabilised power scheme
    (97, 8, 4, 2, 0.0, "wigner"),      # q >= 2 re-orthonormalisation, uneven row blocks
    (120, 12, 4, 1, 0.0, "c3"),        # ill-conditioned sample (CholeskyQR shift policy)
    (80, 10, 5, 1, 0.7, "wigner"),     # Alg. 3 (scaled), shift fused in the local GEMMs
    (60, 3, 2, 0, 0.0, "rank1"),       # rank truncation (basis width 1)
    (96, 10, 6, 1, 0.0, "nearsym"),    # Xᵀ·Y by reduce-scatter (sketch.py:79), even blocks
    (91, 8, 4, 2, 0.0, "nearsym"),     # ... uneven blocks, q = 2
    (90, 8, 4, 1, 0.6, "nearsym"),     # ... scaled: Σ_h (X_hᵀY_h + α S_h)/α
    (96, 10, 6, 1, 0.0, "wigner", "assume"),   # caller-asserted symmetry, no check
    (560, 512, 32, 2, 0.0, "wigner"),  # w = 544 > 512 (C4's k, p, q; two INT8 column groups on GPU)
])
def test_sharded_matches_oracle(tmp_path, case):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    n, k, l, q, alpha, kind = case[:6]
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    assert "error" not in parts[0], str(parts[0]["error"])
    res = np.concatenate([p["rows"] for p in parts], 0)
    x = _matrix(n, kind)
    om = np.random.default_rng(7).standard_normal((n, k + l))
    ref = orc.ran_proj_scal(x, k, l, q, alpha, omega=om) if alpha > 0 else orc.ran_proj(x, k, l, q, omega=om)
    assert int(parts[0]["eff"]) == ref.effective_rank
    assert int(parts[0]["width"]) == ref.basis_width
    want = -1 if len(case) > 6 else (0 if kind == "nearsym" else 1)
    assert all(int(p["bitwise"]) == want for p in parts)   # which Xᵀ branch ran
    err = np.linalg.norm(res - ref.result) / max(np.linalg.norm(ref.result), 1e-300)
    assert err <= 1e-10, err


def test_sharded_rejects_asymmetric(tmp_path):
    """require_symmetric semantics across ranks: the offending pair (5, n−3) sits in
    an off-diagonal block whose mirror lives on the other rank."""
    world = 2
    case = (64, 6, 2, 1, 0.0, "asym")
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert str(np.load(tmp_path / f"r{r}.npz")["error"]) == "AsymmetricMatrixError"
