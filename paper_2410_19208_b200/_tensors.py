"""Host/device plumbing for the reference-shaped API: numpy in → numpy out,
torch CUDA tensor in → torch CUDA tensor out (device resident, no copies)."""

from __future__ import annotations

import numpy as np
import torch

from . import _native, errors


def default_device():
    _native.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


class Operand:
    """A float64 device view of a user matrix plus how to hand results back."""

    __slots__ = ("t", "kind", "device")

    def __init__(self, t, kind, device):
        self.t, self.kind, self.device = t, kind, device

    def give_back(self, t):
        if self.kind == "numpy":
            return t.cpu().numpy()
        if self.kind == "torch_cpu":
            return t.cpu()
        return t


def as_device(x, device=None, dtype=torch.float64):
    """Upload / view ``x`` as a contiguous CUDA tensor of ``dtype`` (np.asarray(x, float) semantics)."""
    _native.require_cuda()
    if isinstance(x, torch.Tensor):
        kind = "torch_cuda" if x.is_cuda else "torch_cpu"
        dev = x.device if x.is_cuda else (torch.device(device) if device else default_device())
        t = x.to(device=dev, dtype=dtype)
        if not t.is_contiguous():
            t = t.contiguous()
        return Operand(t, kind, dev)
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32 if dtype == torch.float32 else float))
    dev = torch.device(device) if device else default_device()
    t = torch.from_numpy(a)
    if t.numel() > (1 << 20):
        t = t.pin_memory()
    return Operand(t.to(dev, non_blocking=False), "numpy", dev)


def require_square(op):
    t = op.t
    if t.dim() != 2 or t.shape[0] != t.shape[1]:
        raise errors.error("NonSquareError", f"expected a square matrix, got shape {tuple(t.shape)}")
    if t.shape[0] < 1:
        raise errors.error("NonSquareError", "matrix dimension must be at least 1")
    return int(t.shape[0])


class DeviceRng:
    """Counter-based N(0,1) stream generated on the GPU (Philox4x32-10).

    Not the reference's numpy stream: use it when throughput matters more
    than reproducing ``numpy.random.default_rng(seed)`` draws (benchmarks,
    long solver runs).  Parity runs pass a numpy Generator instead.
    """

    def __init__(self, seed=0):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.offset = 0

    def normal(self, shape, device):
        rows, cols = (shape, 1) if isinstance(shape, int) else shape
        out = torch.empty((rows, cols) if not isinstance(shape, int) else (rows,),
                          dtype=torch.float64, device=device)
        lib = _native.load_library()
        _native.check(lib.psd_fill_gaussian(_native.ptr(out), rows, cols, cols, self.seed,
                                            self.offset, _native.stream_handle(device)))
        self.offset += (rows * cols + 1) // 2
        return out


def draw_gaussian(rng, shape, device):
    """Ω / start vectors: numpy Generator draws on the host exactly like the
    reference (symmetric.py:135, sketch.py:106), or DeviceRng draws on device."""
    if isinstance(rng, DeviceRng):
        return rng.normal(shape, device)
    g = rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)
    host = g.standard_normal(shape)
    t = torch.from_numpy(np.ascontiguousarray(host))
    if t.numel() > (1 << 20):
        t = t.pin_memory()
    return t.to(device)
