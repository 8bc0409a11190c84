"""FP64 n×n products emulated on the INT8 tensor cores (Ozaki scheme II,
csrc/ozaki.cu) — the default engine of the FP64 sketch products.

The emulation represents row i of A as integers a_ik·2^(53−e_i) (e_i the
row's max exponent) and column j of P likewise, so each product term is exact
to 2^-53 of its row/column maximum and the INT8 sums are exact integers; the
per-entry error bound used below is therefore K·2^-52·max_k|a_ik|·max_k|p_kj|.
The projection-level parity (≤1e-10 relative Frobenius vs the reference) is
checked by the whole FP64 suite, which runs on this engine by default; here the
engine is compared with the DMMA engine and the GEMM with torch's fp64 GEMM.
"""

import os

import numpy as np
import pytest
import torch

from oracle import psd_oracle as orc

pytestmark = pytest.mark.gpu

# PSD_FP64_OZAKI=0 switches the INT8 engine off process-wide (the DMMA-only run of the suite)
int8_enabled = pytest.mark.skipif(os.environ.get("PSD_FP64_OZAKI", "") == "0",
                                  reason="INT8 engine disabled by PSD_FP64_OZAKI=0")


@pytest.fixture(scope="module")
def ours():
    import paper_2410_19208_b200 as m
    m._native.load_library()
    return m


def _oz(ours, a, p):
    lib = ours._native.load_library()
    m, k = a.shape
    n = p.shape[1]
    c = torch.full((m, n), float("nan"), dtype=torch.float64, device=a.device)
    ours._native.check(lib.psd_gemm_f64_ozaki(ours._native.ptr(a), a.stride(0), ours._native.ptr(p),
                                              p.stride(0), m, n, k, ours._native.ptr(c), c.stride(0),
                                              ours._native.stream_handle(a.device)))
    torch.cuda.synchronize()
    return c


def _bound(a, p):
    k = a.shape[1]
    ra = a.abs().amax(dim=1, keepdim=True)
    cp = p.abs().amax(dim=0, keepdim=True)
    return k * 2.0 ** -52 * ra * cp


@pytest.mark.parametrize("m,n,k", [(256, 16, 128), (300, 40, 200), (1000, 272, 1000), (513, 37, 4099),
                                   (64, 512, 300), (130, 264, 4096), (7, 1, 1), (192, 40, 640), (77, 272, 1024)])
def test_gemm_matches_fp64(ours, m, n, k):
    g = torch.Generator(device="cpu").manual_seed(m * 7 + n + k)
    a = torch.randn(m, k, generator=g, dtype=torch.float64).cuda()
    p = torch.randn(k, n, generator=g, dtype=torch.float64).cuda()
    a[::5] *= 1e-7
    p[:, ::3] *= 1e5
    c = _oz(ours, a, p)
    ref = a @ p
    assert not c.isnan().any()
    assert bool(((c - ref).abs() <= _bound(a, p) + 1e-15 * ref.abs()).all())
    assert float((c - ref).norm() / ref.norm()) < 1e-14


@pytest.mark.parametrize("k", [2048, 2040])
def test_gemm_integer_inputs_exact(ours, k):
    g = torch.Generator(device="cpu").manual_seed(3)
    a = torch.randint(-2 ** 20, 2 ** 20, (384, k), generator=g, dtype=torch.int64)
    p = torch.randint(-2 ** 20, 2 ** 20, (k, 96), generator=g, dtype=torch.int64)
    ref = a @ p                        # |entries| < 2^51: exact in fp64
    c = _oz(ours, a.double().cuda(), p.double().cuda())
    assert torch.equal(c.cpu(), ref.double())


@pytest.mark.parametrize("k", [640, 650])   # k % 64 == 0: byte-MMA residues; else the fp32-limb kernel
def test_gemm_zero_rows_extreme_scales(ours, k):
    g = torch.Generator(device="cpu").manual_seed(5)
    a = torch.randn(200, k, generator=g, dtype=torch.float64)
    p = torch.randn(k, 48, generator=g, dtype=torch.float64)
    a[3] = 0.0
    a[4] *= 1e-300
    a[5] *= 1e300
    p[:, 7] = 0.0
    p[:, 8] *= 1e-200
    a, p = a.cuda(), p.cuda()
    c = _oz(ours, a, p)
    ref = a @ p
    assert torch.equal(c[3], torch.zeros_like(c[3])) and torch.equal(c[:, 7], torch.zeros_like(c[:, 7]))
    assert bool(((c - ref).abs() <= _bound(a, p) + 1e-15 * ref.abs()).all())


def test_gemm_long_k_multiple_splits(ours):
    # K > 32768 forces ≥ 2 K-splits (the INT8 sums of one split stay below 2^29)
    g = torch.Generator(device="cpu").manual_seed(9)
    a = torch.randn(256, 40000, generator=g, dtype=torch.float64).cuda()
    p = torch.randn(40000, 24, generator=g, dtype=torch.float64).cuda()
    c = _oz(ours, a, p)
    ref = a @ p
    assert bool(((c - ref).abs() <= _bound(a, p) + 1e-15 * ref.abs()).all())


def _int8_stream(ours, a, p, alpha=0.0, s=None, chunk=0):
    import ctypes
    lib = ours._native.load_library()
    m, k = a.shape
    n = p.shape[1]
    nb = ctypes.c_int64(0)
    ours._native.check(lib.psd_gemm_f64_int8_ws_bytes(m, n, k, chunk, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=a.device)
    c = torch.full((m, n), float("nan"), dtype=torch.float64, device=a.device)
    ours._native.check(lib.psd_gemm_f64_int8(
        ours._native.ptr(a), a.stride(0), ours._native.ptr(p), p.stride(0), m, n, k, ours._native.ptr(c),
        c.stride(0), alpha, ours._native.ptr(s) if s is not None else None, s.stride(0) if s is not None else 0,
        ours._native.ptr(ws), ws.numel(), chunk, ours._native.stream_handle(a.device)))
    torch.cuda.synchronize()
    return c


@pytest.mark.parametrize("m,n,k,chunk", [(350, 40, 300, 100), (1000, 272, 777, 256), (64, 17, 33000, 0),
                                         (300, 544, 600, 128), (90, 1100, 200, 0)])
def test_streamed_general_gemm(ours, m, n, k, chunk):
    """General (non-symmetric) A streamed in row chunks, panel prepared once."""
    g = torch.Generator(device="cpu").manual_seed(m + n + k)
    a = torch.randn(m, k, generator=g, dtype=torch.float64).cuda()
    p = torch.randn(k, n, generator=g, dtype=torch.float64).cuda()
    a[::3] *= 1e4
    c = _int8_stream(ours, a, p, chunk=chunk)
    ref = a @ p
    assert bool(((c - ref).abs() <= _bound(a, p) + 1e-15 * ref.abs()).all())


def test_streamed_gemm_shift_epilogue(ours):
    """(A·P + α·S)/α — the B = (X + αI)/α product of Alg. 3 on a row block."""
    g = torch.Generator(device="cpu").manual_seed(77)
    a = torch.randn(300, 500, generator=g, dtype=torch.float64).cuda()
    p = torch.randn(500, 24, generator=g, dtype=torch.float64).cuda()
    s = p[100:400]
    c = _int8_stream(ours, a, p, alpha=0.75, s=s, chunk=128)
    ref = (a @ p + 0.75 * s) / 0.75
    assert float((c - ref).norm() / ref.norm()) < 1e-14


def test_streamed_gemm_workspace_too_small(ours):
    import ctypes
    lib = ours._native.load_library()
    a = torch.randn(64, 64, dtype=torch.float64).cuda()
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    c = torch.empty(64, 8, dtype=torch.float64, device="cuda")
    st = lib.psd_gemm_f64_int8(ours._native.ptr(a), 64, ours._native.ptr(a), 64, 64, 8, 64, ours._native.ptr(c), 8,
                               0.0, None, 0, ours._native.ptr(ws), 16, 0, ours._native.stream_handle(a.device))
    assert st == 1 and b"workspace" in lib.psd_last_error()


def _sym(n, seed):
    x = np.random.default_rng(seed).standard_normal((n, n))
    return (x + x.T) / 2


@int8_enabled
@pytest.mark.parametrize("q", [0, 1, 2])
def test_ran_proj_int8_engine_matches_dmma_and_oracle(ours, q):
    x = _sym(600, 11 + q)
    params = ours.RangeParams(k=40, l=8, q=q)
    prev = ours.set_fp64_engine("int8")
    try:
        r8 = ours.ran_proj(x, params, np.random.default_rng(5))
        ours.set_fp64_engine("dmma")
        rd = ours.ran_proj(x, params, np.random.default_rng(5))
    finally:
        ours.set_fp64_engine(prev)
    assert r8.device_info["sketch_engine"] == 1 and rd.device_info["sketch_engine"] == 0
    if os.environ.get("PSD_OZ_SYRK", "") != "0":   # PSD_OZ_SYRK=0 keeps the DMMA reconstruction
        assert r8.device_info["recon_engine"] == 1 and rd.device_info["recon_engine"] == 0
    ref = orc.ran_proj(x, 40, 8, q, rng=np.random.default_rng(5)).result
    for r in (r8, rd):
        assert np.linalg.norm(r.result - ref) / np.linalg.norm(ref) < 1e-10
    assert np.linalg.norm(r8.result - rd.result) / np.linalg.norm(rd.result) < 1e-12


@int8_enabled
def test_ran_proj_scal_int8_engine(ours):
    x = _sym(520, 21)
    params = ours.RangeParams(k=30, l=10, q=1)
    prev = ours.set_fp64_engine("int8")
    try:
        r8 = ours.ran_proj_scal(x, params, 0.75, np.random.default_rng(2))
    finally:
        ours.set_fp64_engine(prev)
    assert r8.device_info["sketch_engine"] == 1
    ref = orc.ran_proj_scal(x, 30, 10, 1, 0.75, rng=np.random.default_rng(2)).result
    assert np.linalg.norm(r8.result - ref) / np.linalg.norm(ref) < 1e-10


@int8_enabled
def test_wide_sketch_column_groups_and_transpose_on_dmma(ours):
    x = _sym(700, 4)
    prev = ours.set_fp64_engine("int8")
    try:
        wide = ours.ran_proj(x, ours.RangeParams(k=500, l=16, q=0), np.random.default_rng(1))
        y = x.copy()
        y[0, 1] += 1e-14                                    # not bitwise symmetric → Xᵀ·P kernel
        t = ours.ran_proj(y, ours.RangeParams(k=20, l=8, q=1), np.random.default_rng(1))
    finally:
        ours.set_fp64_engine(prev)
    assert wide.device_info["sketch_engine"] == 1          # w = 516 > 512: two column groups
    ref = orc.ran_proj(x, 500, 16, 0, rng=np.random.default_rng(1)).result
    assert np.linalg.norm(wide.result - ref) / np.linalg.norm(ref) < 1e-10
    assert t.device_info["sketch_engine"] == 3 and t.device_info["used_transpose"] == 1
    ref = orc.ran_proj(y, 20, 8, 1, rng=np.random.default_rng(1)).result
    assert np.linalg.norm(t.result - ref) / np.linalg.norm(ref) < 1e-10


def test_set_fp64_engine_validation(ours):
    with pytest.raises(Exception):
        ours.set_fp64_engine("fp16")


@int8_enabled
def test_auto_engine_size_threshold(ours):
    """auto: DMMA below n = 3072 (measured crossover), INT8 emulation from there."""
    assert ours.set_fp64_engine("auto") in ("auto", "int8", "dmma")
    small = ours.ran_proj(_sym(600, 3), ours.RangeParams(k=20, l=6, q=0), np.random.default_rng(0))
    assert small.device_info["sketch_engine"] == 0
    xs = torch.randn(3072, 3072, dtype=torch.float64, device="cuda")
    xs = (xs + xs.T) / 2
    big = ours.ran_proj(xs, ours.RangeParams(k=20, l=6, q=0), np.random.default_rng(0))
    assert big.device_info["sketch_engine"] == 1
