"""Kernel-level GPU tests: the FP64 DMMA GEMM in every layout / epilogue
against a torch fp64 reference, the symmetric eigensolver, the Philox
Gaussian fill and the symmetry-statistics pass."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2410_19208_b200 as psd
    lib = psd._native.load_library()
    return torch, psd, lib


def _gemm(env, a_layout, b_layout, A, B, M, N, K, epi=0, alpha=1.0, S=None, ws=True, C=None):
    torch, psd, lib = env
    dev = A.device
    if C is None:
        C = torch.full((M, N), np.nan, dtype=torch.float64, device=dev)
    wsb = torch.empty(64 * max(M, 1) * (N + 1) + (1 << 20), dtype=torch.float64, device=dev) if ws else None
    st = psd._native.check(lib.psd_gemm_f64(
        a_layout, b_layout, psd._native.ptr(A), A.stride(0), psd._native.ptr(B), B.stride(0),
        psd._native.ptr(C), C.stride(0), M, N, K, epi, alpha,
        psd._native.ptr(S) if S is not None else ctypes.c_void_p(0), S.stride(0) if S is not None else 0,
        psd._native.ptr(wsb) if wsb is not None else ctypes.c_void_p(0), wsb.numel() if wsb is not None else 0,
        psd._native.stream_handle(dev)))
    torch.cuda.synchronize()
    return C


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 288, 16), (200, 272, 1000),
                                   (1000, 50, 1000), (333, 544, 257), (130, 9, 4099)])
@pytest.mark.parametrize("al,bl", [(0, 0), (1, 0), (0, 1)])
def test_gemm_layouts(env, M, N, K, al, bl):
    torch = env[0]
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    a = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    A = a if al == 0 else a.T.contiguous()
    B = b if bl == 0 else b.T.contiguous()
    C = _gemm(env, al, bl, A, B, M, N, K)
    ref = a @ b
    err = (C - ref).abs().max().item() / max(ref.abs().max().item(), 1e-300)
    assert err < 1e-13, err


def test_gemm_odd_leading_dimensions(env):
    torch = env[0]
    base = torch.randn(301, 303, dtype=torch.float64, device="cuda")
    A = base[:, :77]             # lda = 303 (odd) → 8-byte cp.async path
    B = torch.randn(77, 41, dtype=torch.float64, device="cuda")
    C = _gemm(env, 0, 0, A, B, 301, 41, 77)
    assert (C - A @ B).abs().max().item() < 1e-12


def test_gemm_shift_and_sub_epilogues(env):
    torch = env[0]
    n, w = 513, 40
    X = torch.randn(n, n, dtype=torch.float64, device="cuda")
    P = torch.randn(n, w, dtype=torch.float64, device="cuda")
    alpha = 0.37
    C = _gemm(env, 0, 0, X, P, n, w, n, epi=1, alpha=alpha, S=P)
    ref = (X @ P + alpha * P) / alpha
    assert ((C - ref).abs().max() / ref.abs().max()).item() < 1e-13
    S = torch.randn(n, w, dtype=torch.float64, device="cuda")
    C2 = _gemm(env, 0, 0, X, P, n, w, n, epi=2, S=S, ws=False)
    assert ((C2 - (S - X @ P)).abs().max()).item() < 1e-11


def test_gemm_mirrored_store_is_exactly_symmetric(env):
    torch = env[0]
    n, r = 700, 37
    W = torch.randn(n, r, dtype=torch.float64, device="cuda")
    d = torch.rand(r, dtype=torch.float64, device="cuda")
    WD = W * d
    C = _gemm(env, 0, 1, WD, W, n, n, r, epi=3, ws=False)
    assert torch.equal(C, C.T)
    ref = WD @ W.T
    assert ((C - ref).abs().max() / ref.abs().max()).item() < 1e-13


@pytest.mark.parametrize("m", [1, 2, 17, 50, 64, 144, 272])
def test_eigh_vs_lapack(env, m):
    torch, psd, _ = env
    rng = np.random.default_rng(m)
    g = rng.standard_normal((m, m))
    a = (g + g.T) / 2
    dec = psd.eigh(a)
    ref = np.linalg.eigvalsh(a)[::-1]
    np.testing.assert_allclose(dec.values, ref, atol=1e-12 * max(1, np.abs(ref).max()))
    v = dec.vectors
    assert np.abs(v.T @ v - np.eye(m)).max() < 1e-12 * m
    assert np.abs(v @ np.diag(dec.values) @ v.T - a).max() < 1e-12 * m
    # sign convention: largest-|entry| of each column is positive
    idx = np.argmax(np.abs(v), axis=0)
    assert np.all(v[idx, np.arange(m)] > 0)


def test_eigh_clustered_and_degenerate(env):
    torch, psd, _ = env
    rng = np.random.default_rng(5)
    q, _ = np.linalg.qr(rng.standard_normal((120, 120)))
    lam = np.concatenate([np.full(40, 2.0), np.full(40, -1.0), 1e-14 * rng.standard_normal(40)])
    a = (q * lam) @ q.T
    a = (a + a.T) / 2
    dec = psd.eigh(a)
    np.testing.assert_allclose(np.sort(dec.values), np.sort(np.linalg.eigvalsh(a)), atol=1e-13)
    assert np.abs(dec.vectors @ np.diag(dec.values) @ dec.vectors.T - a).max() < 1e-12


def test_gaussian_fill_statistics(env):
    torch, psd, _ = env
    g = psd.DeviceRng(123)
    x = g.normal((1000, 1000), torch.device("cuda"))
    m, v = x.mean().item(), x.var().item()
    assert abs(m) < 0.01 and abs(v - 1) < 0.01
    y = psd.DeviceRng(123).normal((1000, 1000), torch.device("cuda"))
    assert torch.equal(x, y)


def test_require_symmetric_stats(env):
    torch, psd, _ = env
    rng = np.random.default_rng(3)
    g = rng.standard_normal((333, 333))
    a = (g + g.T) / 2
    assert psd.require_symmetric(a) is not None
    b = a.copy()
    b[5, 7] += 1e-6
    with pytest.raises(psd.AsymmetricMatrixError):
        psd.require_symmetric(b)
    c = a.copy()
    c[5, 7] += 1e-12 * np.abs(a).max()   # within tolerance: accepted
    op = psd._tensors.as_device(c)
    st = psd.symmetric.check_symmetric_device(op)
    assert not st.bitwise and st.defect == pytest.approx(abs(c[5, 7] - c[7, 5]))
    assert st.max_abs == np.abs(c).max()


def test_mirrored_syrk_deterministic_tma_path():
    """The staged-epilogue SYRK (TMA path: even leading dimension) must be
    bitwise reproducible and bitwise symmetric over repeated launches (a
    consumer/store-warp handshake race once produced stale rows)."""
    import torch
    import paper_2410_19208_b200 as psd
    n, r = 1536, 159
    g = torch.Generator(device="cuda").manual_seed(3)
    w = torch.randn(n, r + 1, dtype=torch.float64, device="cuda", generator=g)[:, :r]
    d = torch.rand(r, dtype=torch.float64, device="cuda", generator=g)
    lib = psd._native.load_library()
    plan = psd._native.get_plan(n, r, torch.device("cuda"))

    def recon():
        out = torch.empty((n, n), dtype=torch.float64, device="cuda")
        psd._native.check(lib.psd_reconstruct(plan.handle, psd._native.ptr(w), n, w.stride(0),
                                              psd._native.ptr(d), r, psd._native.ptr(out), n,
                                              psd._native.stream_handle(torch.device("cuda"))))
        return out
    ref = recon()
    exact = (w * d) @ w.T
    assert torch.equal(ref, ref.T)
    assert float((ref - exact).abs().max() / exact.abs().max()) < 1e-13
    for _ in range(30):
        assert torch.equal(recon(), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [256, 4096])
def test_symmetric_alpha_estimate_matches_row_gemv(n):
    """min_eig_magnitude (Alg. 5, sketch.py:117-129) with the lower-triangle products of a
    bitwise-symmetric X (psd_min_eig_magnitude_ex) against the row-GEMV chains on the same
    start vectors, and against the CPU oracle."""
    import torch
    import paper_2410_19208_b200 as psd
    from paper_2410_19208_b200._tensors import as_device
    from paper_2410_19208_b200.sketch import min_eig_magnitude_device
    from oracle import psd_oracle as orc
    x = orc.wigner(n, seed=7) + 0.3 * np.eye(n)
    g = np.random.default_rng(3)
    v1, v2 = g.standard_normal(n), g.standard_normal(n)
    op = as_device(torch.from_numpy(x).cuda())
    a = min_eig_magnitude_device(op, 10, None, v1=v1, v2=v2, bitwise_symmetric=True)
    b = min_eig_magnitude_device(op, 10, None, v1=v1, v2=v2, bitwise_symmetric=False)
    ref = orc.min_eig_magnitude(x, 10, v1=v1, v2=v2)
    assert abs(a - b) <= 1e-12 * max(1.0, abs(b))
    assert abs(a - ref) <= 1e-10 * max(1.0, abs(ref))


@pytest.mark.gpu
def test_power_step_qr_redo_path():
    """q = 2 on a graded spectrum: the power-step samples are ill-conditioned (κ ≫ 1e4), so a
    device-decided one-pass QR raises its flag and the range finder is redone with the
    host-driven loop (api.cu, kSpanRedo); the result must match the CPU oracle."""
    import paper_2410_19208_b200 as psd
    from oracle import psd_oracle as orc
    n, k, l, q = 512, 24, 8, 2
    g = np.random.default_rng(11)
    u, _ = np.linalg.qr(g.standard_normal((n, n)))
    lam = np.concatenate([np.geomspace(1e4, 1e-4, 20), -np.geomspace(1e2, 1e-3, 20), np.zeros(n - 40)])
    x = (u * lam) @ u.T
    x = (x + x.T) / 2
    om = g.standard_normal((n, k + l))
    rep = psd.ran_proj(x, psd.RangeParams(k=k, l=l, q=q), None, omega=om)
    ref = orc.ran_proj(x, k, l, q, omega=om)
    assert rep.basis_width == ref.basis_width and rep.effective_rank == ref.effective_rank
    err = np.linalg.norm(rep.result - ref.result) / np.linalg.norm(ref.result)
    assert err <= 1e-10, err
