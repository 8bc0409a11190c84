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
        n, k, l, q, alpha, kind = case
        x = orc.wigner(n, seed=3) if kind == "wigner" else orc.c3_matrix(n, seed=4, rank=20)
        if kind == "rank1":
            u = np.random.default_rng(5).standard_normal(n)
            x = np.outer(u, u)
        om = np.random.default_rng(7).standard_normal((n, k + l))
        starts = row_split(n, world)
        r0, r1 = starts[rank], starts[rank + 1]
        rep = sharded_ran_proj(torch.from_numpy(x[r0:r1].copy()), r0, n, torch.from_numpy(om),
                               RangeParams(k=k, l=l, q=q), alpha=alpha, comm=Comm(), ops=NumpyOps())
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), rows=rep.result_rows.numpy(), r0=r0, r1=r1,
                 eff=rep.effective_rank, width=rep.basis_width)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (96, 10, 6, 1, 0.0, "wigner"),     # unstabilised power scheme
    (97, 8, 4, 2, 0.0, "wigner"),      # q >= 2 re-orthonormalisation, uneven row blocks
    (120, 12, 4, 1, 0.0, "c3"),        # ill-conditioned sample (CholeskyQR shift policy)
    (80, 10, 5, 1, 0.7, "wigner"),     # Alg. 3 (scaled), shift fused in the local GEMMs
    (60, 3, 2, 0, 0.0, "rank1"),       # rank truncation (basis width 1)
])
def test_sharded_matches_oracle(tmp_path, case):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    n, k, l, q, alpha, kind = case
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    res = np.concatenate([p["rows"] for p in parts], 0)
    x = orc.wigner(n, seed=3) if kind == "wigner" else orc.c3_matrix(n, seed=4, rank=20)
    if kind == "rank1":
        u = np.random.default_rng(5).standard_normal(n)
        x = np.outer(u, u)
    om = np.random.default_rng(7).standard_normal((n, k + l))
    ref = orc.ran_proj_scal(x, k, l, q, alpha, omega=om) if alpha > 0 else orc.ran_proj(x, k, l, q, omega=om)
    assert int(parts[0]["eff"]) == ref.effective_rank
    assert int(parts[0]["width"]) == ref.basis_width
    err = np.linalg.norm(res - ref.result) / max(np.linalg.norm(ref.result), 1e-300)
    assert err <= 1e-10, err
