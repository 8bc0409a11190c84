"""Streaming many host-resident projections through one GPU.

A user of the reference projects matrices one at a time (``ran_proj`` /
``ran_proj_scal``, projection.py:92-159); with host matrices every call pays
the host→device upload of X and the device→host download of X̂₊ (8n² bytes
each way, PCIe-bound at BASELINE config 3).  ``ran_proj_many`` keeps the
per-matrix semantics — same validation, same Ω draw order from ``rng``, one
ProjectionReport per input — but double-buffers X and the result on the
device and runs the copies on two side streams, so the upload of X_{i+1} and
the download of X̂₊_{i−1} proceed (PCIe is full duplex) while X_i is
projected on the caller's stream.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import errors
from .projection import ran_proj, ran_proj_scal, resolve_dtype
from ._tensors import default_device


# PSD_PIPE_STAGGER=1: start X_i's projection only after the download of X̂₊_{i−1}
# finished (kept as an option; tools/probe_e2e.py at C3 on the B200 box, round 1:
# staggered 3.62 projections/s, fully overlapped 4.70/s over 8 steps — both copy
# directions then run at ≈45 GB/s each for the whole step and the 30 ms projection
# hides under them).
_STAGGER = os.environ.get("PSD_PIPE_STAGGER", "0") == "1"


def _host_tensor(x, dtype):
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            raise errors.error("InvalidParams", "ran_proj_many streams HOST matrices; got a CUDA tensor")
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=float)))
    if t.dim() != 2 or t.shape[0] != t.shape[1]:
        raise errors.error("NonSquareError", f"expected a square matrix, got shape {tuple(t.shape)}")
    if t.dtype != dtype:
        t = t.to(dtype)
    return t if t.is_contiguous() else t.contiguous()


def ran_proj_many(xs, params, rng, *, alpha=None, out=None, dtype=None, assume_symmetric=False,
                  device=None):
    """Project every host matrix in ``xs`` (Alg. 2, or Alg. 3 when ``alpha`` is given).

    ``xs``: sequence of square host matrices (torch CPU tensors — pinned for
    full PCIe rate — or numpy arrays), all of one size.  ``out``: optional
    sequence of host tensors receiving the projections (allocated pinned if
    omitted).  Returns the ProjectionReports in input order, ``result`` being
    the host tensor (numpy array for numpy inputs)."""
    xs = list(xs)
    if not xs:
        return []
    tdtype = torch.float32 if resolve_dtype(dtype) == "fp32" else torch.float64
    hosts = [_host_tensor(x, tdtype) for x in xs]
    n = hosts[0].shape[0]
    if any(h.shape[0] != n for h in hosts):
        raise errors.error("DimensionMismatch", "ran_proj_many needs matrices of one size")
    numpy_in = not isinstance(xs[0], torch.Tensor)
    dev = torch.device(device) if device is not None else default_device()
    if out is None:
        out = [torch.empty((n, n), dtype=tdtype, pin_memory=True) for _ in hosts]
    elif len(out) != len(hosts):
        raise errors.error("DimensionMismatch", "out must hold one matrix per input")
    compute = torch.cuda.current_stream(dev)
    up = torch.cuda.Stream(dev)
    down = torch.cuda.Stream(dev)
    nb = min(2, len(hosts))
    xbuf = [torch.empty((n, n), dtype=tdtype, device=dev) for _ in range(nb)]
    rbuf = [torch.empty((n, n), dtype=tdtype, device=dev) for _ in range(nb)]
    uploaded = [torch.cuda.Event() for _ in range(nb)]
    consumed = [None] * nb               # compute finished reading xbuf[s]
    downloaded = [None] * nb             # download of rbuf[s] finished

    def upload(i):
        s = i % len(xbuf)
        with torch.cuda.stream(up):
            if consumed[s] is not None:
                up.wait_event(consumed[s])
            xbuf[s].copy_(hosts[i], non_blocking=True)
            uploaded[s].record(up)

    reports = []
    upload(0)
    for i in range(len(hosts)):
        s = i % len(xbuf)
        if i + 1 < len(hosts):
            upload(i + 1)                # overlaps the projection of X_i
        compute.wait_event(uploaded[s])
        prev = downloaded[(i - 1) % len(xbuf)] if i > 0 else None
        if prev is not None and _STAGGER:
            compute.wait_event(prev)
        if downloaded[s] is not None:
            compute.wait_event(downloaded[s])
        if alpha is None:
            rep = ran_proj(xbuf[s], params, rng, assume_symmetric=assume_symmetric, dtype=tdtype,
                           out=rbuf[s])
        else:
            rep = ran_proj_scal(xbuf[s], params, alpha, rng, assume_symmetric=assume_symmetric,
                                dtype=tdtype, out=rbuf[s])
        done = torch.cuda.Event()
        done.record(compute)
        consumed[s] = done
        with torch.cuda.stream(down):
            down.wait_event(done)
            out[i].copy_(rbuf[s], non_blocking=True)   # overlaps the next upload and projection
            ev = torch.cuda.Event()
            ev.record(down)
            downloaded[s] = ev
        rep.result = out[i]
        reports.append(rep)
    down.synchronize()
    if numpy_in:
        for rep in reports:
            rep.result = rep.result.numpy()
    return reports


__all__ = ["ran_proj_many"]
