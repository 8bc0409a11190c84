"""Row-block sharded randomized PSD projection across the GPUs of one node
(BASELINE config 4).

Rank g owns X_g = X[rows_g, :] (n/G × n).  Every n×n product is rank-local
once its n×w panel has been gathered; the only exchanges are

* ``all_gather`` of the n×w panel before each power-scheme multiply and
  before the compression (Y → Z → Y → Q), and
* ``all_reduce`` (sum) of the w×w Gram matrices of the distributed
  CholeskyQR passes and of T = Σ_g Q_gᵀ (X_g Q),

exactly the exchanges of the reference algorithm's data flow
(sketch.py:75-93, projection.py:101-107).  The k×k eigen-decomposition is
replicated (identical all-reduced T on every rank ⇒ identical eigenpairs).
Rank g returns its row block X̂₊[rows_g, :] = (W_g·D)·Wᵀ.

Symmetry.  ``symmetric="check"`` (the default) runs the
reference's ``require_symmetric`` (symmetric.py:39-57, called at
projection.py:100) on the sharded X: the diagonal block locally and every
off-diagonal block pair (X[rows_g, cols_h], X[rows_h, cols_g]) exchanged
point-to-point in row chunks — one pass over X, ≈ 1/G of it per rank over
NVLink — with a global max|x| / max|x − xᵀ| reduction; an X outside the
tolerance raises ``AsymmetricMatrixError``.  For a bitwise-symmetric X
(every BASELINE config, by construction) (XᵀY)_g = X_g·Y, so the Xᵀ product of
the power scheme (sketch.py:79) is the same all-gather + local GEMM as the X
products.  For an X that is symmetric only within tolerance the Xᵀ product
keeps the reference's semantics: each rank forms the full-height partial
X_gᵀ·Y_g and a reduce-scatter sums Σ_h X_hᵀ Y_h into the row blocks (the same
volume as the all-gather it replaces).  ``symmetric="assume"`` skips the check
for inputs the caller guarantees bitwise symmetric (the C4 generator).

The arithmetic goes through an ``ops`` object: ``KernelOps`` binds the
libpsdproj.so kernels (the product path); tests bind a numpy stand-in to
exercise this host logic on CPU ranks (gloo).  Collectives go through
``torch.distributed`` (NCCL on GPUs, gloo on CPU).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native, errors

RANK_TRUNCATION_FACTOR = 1e-12  # sketch.py:12
U64 = 1.1102230246251565e-16
SYM_TOL_FACTOR = 1e-10          # symmetric.py:16
INT8_MAX_K = 1 << 18            # largest K of the exact INT8 emulation (csrc/ozaki.cu)
SYM_CHUNK_ROWS = 8192           # row chunk of the symmetry-check block exchange


def row_split(n, world):
    """Balanced contiguous row ranges: rank g owns [starts[g], starts[g+1])."""
    base, rem = divmod(n, world)
    sizes = [base + (1 if g < rem else 0) for g in range(world)]
    starts = [0]
    for s in sizes:
        starts.append(starts[-1] + s)
    return starts


class Comm:
    """torch.distributed collectives over row blocks.  Equal row blocks (n
    divisible by the world size, as at C4) gather straight into the n×w panel
    and reduce-scatter straight out of the full-height partial; uneven blocks go
    through one padded staging buffer."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def _sizes(self, starts):
        return [starts[g + 1] - starts[g] for g in range(self.world)]

    def all_gather_rows(self, local, starts):
        """The full panel (n × w) from every rank's row block."""
        if self.world == 1:
            return local
        sizes = self._sizes(starts)
        rows = max(sizes)
        tail = tuple(local.shape[1:])
        if min(sizes) == rows:
            full = local.new_empty((starts[-1],) + tail)
            dist.all_gather_into_tensor(full, local.contiguous(), group=self.group)
            return full
        pad = local.new_zeros((rows,) + tail)
        pad[: local.shape[0]] = local
        staged = local.new_empty((self.world * rows,) + tail)
        dist.all_gather_into_tensor(staged, pad, group=self.group)
        full = local.new_empty((starts[-1],) + tail)
        for g in range(self.world):
            full[starts[g]:starts[g + 1]] = staged[g * rows: g * rows + sizes[g]]
        return full

    def reduce_scatter_rows(self, full, starts):
        """This rank's row block of Σ_ranks full (each rank holds an n × w partial)."""
        if self.world == 1:
            return full
        sizes = self._sizes(starts)
        rows = max(sizes)
        tail = tuple(full.shape[1:])
        out = full.new_empty((rows,) + tail)
        if min(sizes) == rows:
            dist.reduce_scatter_tensor(out, full.contiguous(), op=dist.ReduceOp.SUM, group=self.group)
            return out
        staged = full.new_zeros((self.world * rows,) + tail)
        for g in range(self.world):
            staged[g * rows: g * rows + sizes[g]] = full[starts[g]:starts[g + 1]]
        dist.reduce_scatter_tensor(out, staged, op=dist.ReduceOp.SUM, group=self.group)
        return out[: sizes[self.rank]]

    def exchange(self, send, dst, recv, src):
        """Point-to-point: send ``send`` to rank dst while receiving ``recv`` from src."""
        ops = [dist.P2POp(dist.isend, send, dst, group=self.group),
               dist.P2POp(dist.irecv, recv, src, group=self.group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return recv

    def all_reduce_sum(self, t):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def all_reduce_max(self, t):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t


class KernelOps:
    """The product backend: every operation is a libpsdproj.so kernel."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.lib = _native.load_library()
        self.ws = None
        self.ws8 = None
        self.int8_products = 0     # X_g·P products that ran on the INT8 engine

    def _stream(self):
        return _native.stream_handle(self.device)

    def _ws(self, elems):
        if self.ws is None or self.ws.numel() < elems:
            self.ws = torch.empty(int(elems), dtype=torch.float64, device=self.device)
        return self.ws

    def empty(self, shape):
        return torch.empty(shape, dtype=torch.float64, device=self.device)

    def xmul(self, x_rows, panel, shift_alpha=0.0, shift_src=None):
        """X_g·P for the n-wide products (sketch.py:75/:79/:82, projection.py:104): on the
        INT8 tensor cores as an exact FP64 emulation (X_g streamed in row chunks, panels wider
        than 512 columns in column groups) when the FP64 engine is "int8", else the DMMA GEMM."""
        from . import projection
        m, k = x_rows.shape
        n = panel.shape[1]
        eng = projection._FP64_ENGINE
        use = eng == "int8" or (eng == "auto" and k >= projection.INT8_MIN_N)
        use = use and k <= INT8_MAX_K      # exact CRT needs K ≤ 2^18 (ozaki.cu kMaxK)
        if not use or x_rows.stride(1) != 1 or panel.stride(1) != 1:
            return self.matmul(x_rows, panel, shift_alpha=shift_alpha, shift_src=shift_src)
        out = self.empty((m, n))
        chunk = 8192
        nbytes = ctypes.c_int64(0)
        _native.check(self.lib.psd_gemm_f64_int8_ws_bytes(m, n, k, chunk, ctypes.byref(nbytes)))
        if self.ws8 is None or self.ws8.numel() < nbytes.value:
            self.ws8 = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
        s = shift_src
        alpha = float(shift_alpha) if shift_alpha > 0.0 else 0.0
        _native.check(self.lib.psd_gemm_f64_int8(
            _native.ptr(x_rows), x_rows.stride(0), _native.ptr(panel), panel.stride(0), m, n, k,
            _native.ptr(out), out.stride(0), alpha,
            _native.ptr(s) if (s is not None and alpha > 0.0) else ctypes.c_void_p(0),
            s.stride(0) if (s is not None and alpha > 0.0) else 0,
            _native.ptr(self.ws8), self.ws8.numel(), chunk, self._stream()))
        self.int8_products += 1
        return out

    def matmul(self, a, b, a_trans=False, b_trans=False, shift_alpha=0.0, shift_src=None):
        """op(a)·op(b); shift_alpha > 0: (acc + α·shift_src)/α (B = (X+αI)/α fused)."""
        m = a.shape[1] if a_trans else a.shape[0]
        k = a.shape[0] if a_trans else a.shape[1]
        n = b.shape[0] if b_trans else b.shape[1]
        out = self.empty((m, n))
        epi = 1 if shift_alpha > 0.0 else 0
        ldw = (n + 1) // 2 * 2
        ws = self._ws(min(256 * m * ldw, max(4 * m * ldw, 1 << 22)) + (1 << 16))
        s = shift_src
        _native.check(self.lib.psd_gemm_f64(
            1 if a_trans else 0, 1 if b_trans else 0, _native.ptr(a), a.stride(0),
            _native.ptr(b), b.stride(0), _native.ptr(out), out.stride(0), m, n, k, epi,
            float(shift_alpha) if epi else 1.0,
            _native.ptr(s) if s is not None else ctypes.c_void_p(0), s.stride(0) if s is not None else 0,
            _native.ptr(ws), ws.numel(), self._stream()))
        return out

    def gram(self, a, b=None):
        g = self.matmul(a, a if b is None else b, a_trans=True)
        if b is None or b is a:
            _native.check(self.lib.psd_symmetrize(_native.ptr(g), g.shape[0], g.stride(0), self._stream()))
        return g

    def symmetrize(self, g):
        _native.check(self.lib.psd_symmetrize(_native.ptr(g), g.shape[0], g.stride(0), self._stream()))
        return g

    def chol_inv(self, g, shift):
        m = g.shape[0]
        l_ = self.empty((m, m))
        rinv = self.empty((m, m))
        scratch = self.empty((m, m))
        status = self.empty((4,))
        _native.check(self.lib.psd_chol_inv(_native.ptr(g), m, g.stride(0), float(shift),
                                            _native.ptr(l_), m, _native.ptr(rinv), m,
                                            _native.ptr(scratch), _native.ptr(status), self._stream()))
        st = status.cpu().tolist()
        return l_, rinv, int(st[0]), st[1], st[2], st[3]

    def diag(self, l_):
        return torch.diagonal(l_).clone()

    def eigh(self, t):
        from .symmetric import eigh_device
        from ._tensors import Operand
        return eigh_device(Operand(t.contiguous(), "torch_cuda", self.device), validate=False)

    def scale_columns(self, w, d):
        out = self.empty(tuple(w.shape))
        _native.check(self.lib.psd_scale_columns(_native.ptr(w), w.stride(0), _native.ptr(d),
                                                 _native.ptr(out), out.stride(0), w.shape[0],
                                                 w.shape[1], self._stream()))
        return out

    def syrk_window(self, a, b, r0, r1):
        """Rows [r0, r1) of the exactly symmetric mirror(lower(a·bᵀ)) (n×n)."""
        n = a.shape[0]
        if a.shape[1] % 2 or a.stride(0) % 2:  # TMA needs 16-byte rows: zero-pad the width
            kp = a.shape[1] + 1
            pa, pb = self.empty((n, kp)).zero_(), self.empty((n, kp)).zero_()
            pa[:, : a.shape[1]] = a
            pb[:, : b.shape[1]] = b
            a, b = pa, pb
        out = self.empty((r1 - r0, n))
        _native.check(self.lib.psd_syrk_window(_native.ptr(a), a.stride(0), _native.ptr(b),
                                               b.stride(0), n, a.shape[1], r0, r1,
                                               _native.ptr(out), out.stride(0), self._stream()))
        return out

    def sym_stats(self):
        """Zeroed device accumulator for pair_defect: {max|x|, max defect, flags}."""
        return torch.zeros(3, dtype=torch.float64, device=self.device)

    def pair_defect(self, a, b, stats):
        """Accumulate max|x|, max|a_ij − b_ji| and flags of a block pair."""
        _native.check(self.lib.psd_pair_defect(_native.ptr(a), a.stride(0), _native.ptr(b), b.stride(0),
                                               a.shape[0], a.shape[1], _native.ptr(stats), 0,
                                               self._stream()))
        return stats

    def read_stats(self, stats):
        h = stats.cpu()
        return float(h[0]), float(h[1]), int(h.view(torch.int32)[4])

    def max_abs(self, x):
        out = self.empty((1,))
        _native.check(self.lib.psd_max_abs(_native.ptr(x), x.shape[0], x.shape[1], x.stride(0),
                                           _native.ptr(out), self._stream()))
        return out


@dataclass
class ShardReport:
    result_rows: object      # this rank's row block of X̂₊ (or None)
    row_start: int
    row_stop: int
    effective_rank: int
    basis_width: int
    factors_w_rows: object   # this rank's rows of W (n_g × r₊)
    factors_d: object        # d (r₊), replicated
    alpha_used: float | None = None
    qr_passes: int = 0
    qr_shifted: bool = False
    bitwise_symmetric: bool | None = None   # None: symmetric="assume" (not checked)


def _dist_cholqr(ops, comm, y_loc, starts, n_total, rdiag=None):
    """Distributed CholeskyQR2 / shifted CholeskyQR3 over row blocks; same
    policy as the single-GPU cholqr (api.cu).  Returns (Q_loc, R diag,
    ‖Y‖_F, passes, shifted, zero)."""
    w = y_loc.shape[1]
    cur = y_loc
    rd = torch.ones(w, dtype=torch.float64, device=y_loc.device) if rdiag is not None else None
    unshifted_run, passes, shifted = 0, 0, False
    kest0 = 0.0
    frob = 0.0
    for it in range(10):
        g = comm.all_reduce_sum(ops.gram(cur))
        ops.symmetrize(g)
        if unshifted_run >= 2:
            dev = (g - torch.eye(w, dtype=g.dtype, device=g.device)).abs().max().item()
            if dev <= 1e-13 * max(1, w):
                break
        l_, rinv, info, trace, dmin, dmax = ops.chol_inv(g, 0.0)
        if it == 0:
            frob = math.sqrt(max(trace, 0.0))
            if trace == 0.0:
                return cur, rd, 0.0, passes, shifted, True
        if not math.isfinite(trace):
            raise errors.error("ConvergenceFailure", "non-finite Gram matrix in QR")
        bad = info != 0 or not (math.isfinite(dmin) and math.isfinite(dmax))
        kest = dmax / dmin if dmin > 0 else math.inf
        if it == 0:
            kest0 = kest
        shift = bad or kest > 3e6
        if shift:
            s = 11.0 * (float(n_total) * w + w * (w + 1.0)) * U64 * trace
            l_, rinv, info, _, _, _ = ops.chol_inv(g, s)
            if info != 0:
                raise errors.error("ConvergenceFailure", f"shifted CholeskyQR broke down (pivot {info})")
            shifted = True
        if rd is not None:
            rd = rd * ops.diag(l_).abs()
        cur = ops.matmul(cur, rinv)
        passes += 1
        unshifted_run = 0 if shift else unshifted_run + 1
        if unshifted_run >= 2 and kest0 <= 1e4:
            break
    return cur, rd, frob, passes, shifted, False


def sharded_symmetry_stats(x_rows, row_start, n, comm, ops, chunk_rows=SYM_CHUNK_ROWS):
    """Global (max|x|, max|x − xᵀ|, bitwise, finite) of a row-sharded X: the
    diagonal block locally, every off-diagonal block pair exchanged
    point-to-point (ring schedule: at step s rank g sends X[rows_g, cols_{g+s}]
    to g+s and receives X[rows_{g−s}, cols_g] from g−s), in row chunks of the
    sender so each message is ≤ chunk_rows × n_g doubles."""
    starts = row_split(n, comm.world)
    g = comm.rank
    r0, r1 = starts[g], starts[g + 1]
    stats = ops.sym_stats()
    diag = x_rows[:, r0:r1]
    ops.pair_defect(diag, diag, stats)
    for s in range(1, comm.world):
        dst, src = (g + s) % comm.world, (g - s) % comm.world
        d0, d1 = starts[dst], starts[dst + 1]
        s0, s1 = starts[src], starts[src + 1]
        nchunks = max(math.ceil((r1 - r0) / chunk_rows), math.ceil((s1 - s0) / chunk_rows), 1)
        for c in range(nchunks):
            a0, a1 = min(c * chunk_rows, r1 - r0), min((c + 1) * chunk_rows, r1 - r0)
            b0, b1 = min(c * chunk_rows, s1 - s0), min((c + 1) * chunk_rows, s1 - s0)
            send = x_rows[a0:a1, d0:d1].contiguous()          # X[rows_g chunk, cols_dst]
            recv = x_rows.new_empty((b1 - b0, r1 - r0))       # X[rows_src chunk, cols_g]
            comm.exchange(send, dst, recv, src)
            if b1 > b0:
                # a = X[rows_g, cols_src chunk] (n_g × c), b = X[rows_src chunk, cols_g] (c × n_g)
                ops.pair_defect(x_rows[:, s0 + b0:s0 + b1], recv, stats)
    mx, defect, flags = ops.read_stats(stats)
    red = torch.tensor([mx, defect, float(flags & 1), float((flags >> 1) & 1)], dtype=torch.float64,
                       device=x_rows.device)
    comm.all_reduce_max(red)
    return float(red[0]), float(red[1]), red[2].item() == 0.0, red[3].item() == 0.0


def sharded_ran_proj(x_rows, row_start, n, omega, params, *, alpha=0.0, comm=None, ops=None,
                     want_result=True, strict=False, symmetric="check", tol=None):
    """Alg. 2 (alpha = 0) / Alg. 3 (alpha > 0) on a row-sharded X.

    x_rows: this rank's rows [row_start, row_start + n_g) of X (n_g × n).
    omega:  the full n × (k+l) Gaussian test matrix (identical on all ranks).
    symmetric: "check" — require_symmetric on the sharded X (raises
        AsymmetricMatrixError like projection.py:100); Xᵀ products by
        reduce-scatter unless X is bitwise symmetric.  "assume" — the caller
        guarantees a bitwise-symmetric X; no check.
    """
    comm = comm or Comm()
    ops = ops or KernelOps(x_rows.device)
    starts = row_split(n, comm.world)
    r0, r1 = starts[comm.rank], starts[comm.rank + 1]
    if (r0, r1 - r0) != (row_start, x_rows.shape[0]):
        raise errors.error("DimensionMismatch",
                           f"rank {comm.rank} holds rows [{row_start}, {row_start + x_rows.shape[0]}), "
                           f"expected [{r0}, {r1})")
    width = params.width
    if symmetric not in ("check", "assume"):
        raise errors.error("InvalidParams", f"symmetric must be 'check' or 'assume', got {symmetric!r}")
    bitwise, mx = True, None
    if symmetric == "check":                                    # projection.py:100
        mx, defect, bitwise, finite = sharded_symmetry_stats(x_rows, row_start, n, comm, ops)
        limit = SYM_TOL_FACTOR * max(1.0, mx) if tol is None else float(tol)
        if not finite:
            raise errors.error("ConvergenceFailure", "matrix has non-finite entries")
        if defect > limit:
            raise errors.error("AsymmetricMatrixError",
                               f"matrix is not symmetric: max asymmetry {defect:.3e} exceeds "
                               f"tolerance {limit:.3e}")
    checked = bitwise if symmetric == "check" else None
    if width > n:
        raise errors.error("InvalidParams", f"k+l = {width} exceeds min(m, n) = {n}")
    if alpha > 0.0:  # projection.py:133-137 with a global max|x|
        if mx is None:
            mx = comm.all_reduce_max(ops.max_abs(x_rows)).item()
        alpha_tol = 1e-12 * max(1.0, mx)
        if alpha <= alpha_tol:
            raise errors.error("AlphaTooSmall",
                               f"alpha = {alpha:.3e} is at or below tolerance {alpha_tol:.3e}; input is numerically PSD")

    def xmul(panel_full):
        # (X P)[rows_g] or, scaled, ((X + αI) P / α)[rows_g]
        mul = getattr(ops, "xmul", None) or ops.matmul
        if alpha > 0.0:
            return mul(x_rows, panel_full, shift_alpha=alpha, shift_src=panel_full[r0:r1])
        return mul(x_rows, panel_full)

    def xtmul(y_loc):
        # (Xᵀ Y)_g (sketch.py:79).  Bitwise-symmetric X: X_g·Y after an all-gather.
        # Otherwise Σ_h X_hᵀ Y_h by reduce-scatter; scaled: each rank's partial is
        # (X_hᵀ Y_h + α·S_h)/α with S_h = Y_h in rows_h (zero elsewhere), so the sum
        # is BᵀY = (XᵀY + αY)/α.
        if bitwise:
            return xmul(comm.all_gather_rows(y_loc, starts))
        if alpha > 0.0:
            shift = ops.empty((n, y_loc.shape[1])).zero_()
            shift[r0:r1] = y_loc
            part = ops.matmul(x_rows, y_loc, a_trans=True, shift_alpha=alpha, shift_src=shift)
        else:
            part = ops.matmul(x_rows, y_loc, a_trans=True)
        return comm.reduce_scatter_rows(part, starts)

    stabilize = params.q >= 2                                   # sketch.py:74
    y = xmul(omega)                                             # sketch.py:75
    for _ in range(params.q):                                   # sketch.py:76-82
        if stabilize:
            y = _dist_cholqr(ops, comm, y, starts, n)[0]
        z = xtmul(y)                                            # sketch.py:79
        if stabilize:
            z = _dist_cholqr(ops, comm, z, starts, n)[0]
        y = xmul(comm.all_gather_rows(z, starts))
    q_loc, rd, frob, passes, shifted, zero = _dist_cholqr(ops, comm, y, starts, n, rdiag=True)
    if zero:
        keep = []
    else:
        keep = [i for i, v in enumerate(rd.cpu().tolist()) if v > RANK_TRUNCATION_FACTOR * frob]
    if len(keep) < width:
        if strict:
            raise errors.error("RankDeficientSample",
                               f"sampled matrix has numerical rank {len(keep)} < {width}")
        if keep:
            q_loc = q_loc[:, keep].contiguous()
    wk = len(keep)
    if wk == 0:
        return ShardReport(None if not want_result else ops.empty((r1 - r0, n)).zero_(), r0, r1, 0, 0,
                           ops.empty((r1 - r0, 0)), ops.empty((0,)), alpha if alpha > 0 else None,
                           passes, shifted, checked)
    q_full = comm.all_gather_rows(q_loc, starts)
    c_loc = xmul(q_full)                                        # (X Q)_g or (B Q)_g
    t = comm.all_reduce_sum(ops.gram(q_loc, c_loc))             # Σ_g Q_gᵀ (X Q)_g
    ops.symmetrize(t)                                           # projection.py:104
    vals, vecs = ops.eigh(t)                                    # projection.py:105
    offset = 1.0 if alpha > 0.0 else 0.0
    clipped = vals - offset
    r = int((clipped > 0.0).sum().item())
    scale = alpha if alpha > 0.0 else 1.0
    d = (clipped[:r] * scale).contiguous()
    if r == 0:
        res = ops.empty((r1 - r0, n)).zero_() if want_result else None
        return ShardReport(res, r0, r1, 0, wk, ops.empty((r1 - r0, 0)), d,
                           alpha if alpha > 0 else None, passes, shifted, checked)
    u = vecs[:, :r].contiguous()
    w_loc = ops.matmul(q_loc, u)                                # W_g = Q_g U₊
    res = None
    if want_result:
        # rows_g of sym((W D) Wᵀ) from lower tiles, mirrored: the row blocks of
        # all ranks assemble into a bitwise-symmetric X̂₊ (projection.py:78)
        w_full = comm.all_gather_rows(w_loc, starts)
        res = ops.syrk_window(ops.scale_columns(w_full, d), w_full, r0, r1)
    return ShardReport(res, r0, r1, r, wk, w_loc, d, alpha if alpha > 0 else None, passes, shifted,
                       checked)
