"""ctypes binding of libpsdproj.so (include/psdproj.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing every entry point raises.  Device buffers are torch tensors (torch is
plumbing here: allocation and streams); only raw pointers cross the ABI.
"""

from __future__ import annotations

import ctypes
import os
import threading
from collections import OrderedDict

import torch

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpsdproj.so")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int32_p = ctypes.POINTER(ctypes.c_int32)


class PsdReport(ctypes.Structure):
    _fields_ = [
        ("effective_rank", ctypes.c_int32),
        ("basis_width", ctypes.c_int32),
        ("used_transpose", ctypes.c_int32),
        ("qr_passes", ctypes.c_int32),
        ("qr_shifted", ctypes.c_int32),
        ("eig_sweeps", ctypes.c_int32),
        ("gpu_launches", ctypes.c_int32),
        ("sketch_engine", ctypes.c_int32),
        ("residual_frob", ctypes.c_double),
        ("max_abs", ctypes.c_double),
        ("sym_defect", ctypes.c_double),
        ("alpha_used", ctypes.c_double),
        ("recon_engine", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


STAGES = ("symcheck", "sketch_gemm", "qr", "compress", "eigh", "recon", "diag", "total", "int8_gemm")

FLAG_DIAGNOSTICS = 1
FLAG_STRICT = 2
FLAG_SKIP_SYMCHECK = 4
FLAG_ASSUME_SYMMETRIC = 8
FLAG_FP64_DMMA = 16
FLAG_FP64_INT8 = 32

# name → (restype, argtypes); the full exported surface of include/psdproj.h
SIGNATURES = {
    "psd_last_error": (ctypes.c_char_p, []),
    "psd_version": (ctypes.c_char_p, []),
    "psd_plan_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_int32]),
    "psd_plan_destroy": (None, [ctypes.c_void_p]),
    "psd_plan_bytes": (ctypes.c_int64, [ctypes.c_void_p]),
    "psd_plan_profile": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_double_p, c_int32_p,
                                        ctypes.c_int32]),
    "psd_plan_prefetch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64]),
    "psd_plan_prefetch_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64]),
    "psd_require_symmetric": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_double, c_double_p,
                                             ctypes.c_void_p]),
    "psd_power_iteration": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_double, ctypes.c_void_p,
                                           ctypes.c_int32, c_double_p, ctypes.c_void_p]),
    "psd_min_eig_magnitude": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_int32, c_double_p, ctypes.c_void_p]),
    "psd_min_eig_magnitude_ex": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                                ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                                ctypes.c_int32, ctypes.c_uint32, c_double_p, ctypes.c_void_p]),
    "psd_range_finder": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_double, ctypes.c_uint32, ctypes.c_void_p,
                                        ctypes.c_int64, c_int32_p, ctypes.c_void_p]),
    "psd_eigh": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, c_int32_p,
                                ctypes.c_void_p]),
    "psd_ran_proj": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                    ctypes.c_double, ctypes.c_uint32, ctypes.c_void_p,
                                    ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.POINTER(PsdReport), ctypes.c_void_p]),
    "psd_ran_proj_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_double, ctypes.c_uint32, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.POINTER(PsdReport), ctypes.c_void_p]),
    "psd_gemm_f64_int8_ws_bytes": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                                   ctypes.POINTER(ctypes.c_int64)]),
    "psd_gemm_f64_int8": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]),
    "psd_gemm_f64_ozaki": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p]),
    "psd_syrk_f64_int8": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_void_p]),
    "psd_gemm_tf32x3": (ctypes.c_int, [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_void_p]),
    "psd_reconstruct": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    "psd_symmetrize": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_void_p]),
    "psd_gemm_f64": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                     ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                     ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    "psd_chol_inv": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p]),
    "psd_scale_columns": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int32, ctypes.c_void_p]),
    "psd_max_abs": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "psd_syrk_window": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_void_p]),
    "psd_fill_sym_gaussian": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_void_p]),
    "psd_pair_defect": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                        ctypes.c_void_p]),
    "psd_sdls_assemble": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "psd_sdls_traces": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "psd_sdls_traces_dense": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "psd_sdls_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_int32, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
    "psd_fill_gaussian": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                         ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_void_p]),
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path=LIB_PATH):
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_2410_19208_b200._build` "
                "(nvcc, sm_100a). There is no CPU fallback.")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status):
    if status != 0:
        msg = load_library().psd_last_error().decode(errors="replace")
        errors.raise_for_status(status, msg)


def require_cuda():
    if not torch.cuda.is_available():
        raise errors.error("DeviceError", "a CUDA device (B200, sm_100a) is required; no CPU fallback")


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def stream_handle(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Plan:
    """Device workspace for problems up to (n, width) — psd_plan_create."""

    def __init__(self, n, width, device):
        lib = load_library()
        self.n, self.width, self.device = int(n), int(width), torch.device(device)
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(lib.psd_plan_create(ctypes.byref(handle), self.n, self.width,
                                      self.device.index or 0))
        self.handle = handle
        self.bytes = lib.psd_plan_bytes(handle)

    def profile(self, enable=None, reset=False):
        """Per-stage (ms, count) accumulated since the last reset (psd_plan_profile)."""
        ms = (ctypes.c_double * len(STAGES))()
        cnt = (ctypes.c_int32 * len(STAGES))()
        en = -1 if enable is None else int(bool(enable))
        check(load_library().psd_plan_profile(self.handle, en, ms, cnt, int(reset)))
        return {name: (ms[i], cnt[i]) for i, name in enumerate(STAGES)}

    def close(self):
        if getattr(self, "handle", None):
            load_library().psd_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_plans: "OrderedDict[tuple, Plan]" = OrderedDict()
_plans_lock = threading.Lock()
MAX_PLANS = 2


def get_plan(n, width, device):
    """Cached plan able to hold (n, width) on ``device`` (LRU of MAX_PLANS)."""
    device = torch.device(device)
    key_dev = (device.type, device.index or 0)
    with _plans_lock:
        for key, plan in _plans.items():
            if key[0] == key_dev and plan.n >= n and plan.width >= width:
                _plans.move_to_end(key)
                return plan
        plan = Plan(n, width, device)
        _plans[(key_dev, n, width)] = plan
        while len(_plans) > MAX_PLANS:
            _, old = _plans.popitem(last=False)
            old.close()
        return plan


def free_plans():
    with _plans_lock:
        while _plans:
            _, p = _plans.popitem()
            p.close()
