"""Test-only numpy stand-in for sharded.KernelOps: lets the multi-rank host
logic of paper_2410_19208_b200.sharded run on CPU ranks (gloo).  Never used
by the product path."""

import numpy as np
import torch

from oracle import psd_oracle as orc


def _np(t):
    return t.detach().cpu().numpy()


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))


class NumpyOps:
    def empty(self, shape):
        return torch.empty(shape, dtype=torch.float64)

    def matmul(self, a, b, a_trans=False, b_trans=False, shift_alpha=0.0, shift_src=None):
        A = _np(a).T if a_trans else _np(a)
        B = _np(b).T if b_trans else _np(b)
        c = A @ B
        if shift_alpha > 0.0:
            c = (c + shift_alpha * _np(shift_src)) / shift_alpha
        return _t(c)

    def gram(self, a, b=None):
        return self.matmul(a, a if b is None else b, a_trans=True)

    def symmetrize(self, g):
        a = _np(g)
        g.copy_(_t((a + a.T) / 2.0))
        return g

    def chol_inv(self, g, shift):
        a = _np(g).copy()
        trace = float(np.trace(a))
        a[np.diag_indices_from(a)] += shift
        try:
            l_ = np.linalg.cholesky(a)
            info = 0
        except np.linalg.LinAlgError:
            return _t(np.eye(a.shape[0])), _t(np.eye(a.shape[0])), 1, trace, 0.0, 0.0
        d = np.diag(l_)
        rinv = np.linalg.inv(l_).T
        return _t(l_), _t(rinv), info, trace, float(d.min()), float(d.max())

    def diag(self, l_):
        return torch.diagonal(l_).clone()

    def eigh(self, t):
        dec = orc.eigh(_np(t))
        return _t(dec.values), _t(dec.vectors)

    def scale_columns(self, w, d):
        return _t(_np(w) * _np(d))

    def syrk_window(self, a, b, r0, r1):
        c = _np(a) @ _np(b).T
        low = np.tril(c)
        sym = low + np.tril(low, -1).T
        return _t(sym[r0:r1])

    def max_abs(self, x):
        return _t(np.array([np.abs(_np(x)).max()]))

    def sym_stats(self):
        return [0.0, 0.0, 0]

    def pair_defect(self, a, b, stats):
        A, B = _np(a), _np(b)
        if A.size:
            stats[0] = max(stats[0], float(np.abs(A).max()), float(np.abs(B).max()))
            stats[1] = max(stats[1], float(np.abs(A - B.T).max()))
            stats[2] |= (1 if np.any(A != B.T) else 0) | (0 if np.all(np.isfinite(A)) else 2)
        return stats

    def read_stats(self, stats):
        return float(stats[0]), float(stats[1]), int(stats[2])
