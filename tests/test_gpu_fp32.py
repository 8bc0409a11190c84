"""FP32 path (BASELINE config 3 "fp32"): 3xTF32 tcgen05 GEMMs with TMEM
accumulators, FP64 QR/eigh, always re-orthonormalised power scheme.

Parity rule (BASELINE north_star): relative Frobenius error
≤ 1e-4 against the FP64 oracle run on the fp32-rounded X and Ω upcast to f64,
so only the arithmetic differs.
"""

import numpy as np
import pytest
import torch

from oracle import psd_oracle as orc
from tests import golden_io as gio

pytestmark = pytest.mark.gpu

TOL32 = 1e-4


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a))


@pytest.fixture(scope="module")
def ours():
    import paper_2410_19208_b200 as m
    m._native.load_library()
    return m


def _gemm(ours, mode, a, b, c):
    lib = ours._native.load_library()
    dev = a.device
    ours._native.check(lib.psd_gemm_tf32x3(mode, ours._native.ptr(a), a.stride(0), ours._native.ptr(b),
                                           b.stride(0), a.shape[0], b.shape[0], a.shape[1],
                                           ours._native.ptr(c), c.stride(0),
                                           ours._native.stream_handle(dev)))


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (128, 16, 16), (127, 17, 33), (256, 48, 64),
                                   (1000, 272, 4096), (300, 520, 1000), (513, 600, 7)])
def test_tf32x3_gemm_matches_fp64(ours, m, n, k):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    a = torch.randn(m, k, device="cuda", generator=g)
    b = torch.randn(n, k, device="cuda", generator=g)
    c = torch.full((m, n), float("nan"), device="cuda", dtype=torch.float64)
    _gemm(ours, 0, a, b, c)
    ref = a.double() @ b.double().T
    err = ((c - ref).norm() / ref.norm()).item()
    # 3xTF32 with FP32 accumulation: the error of an FP32 GEMM, ~√K·2⁻²⁴
    assert err <= 2e-7 * max(1.0, np.sqrt(k)), err


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (256, 48, 64), (1000, 272, 4096), (300, 520, 1000),
                                   (513, 17, 7), (2048, 272, 32768)])
def test_tf32x3_gemm_a_transposed(ours, m, n, k):
    """mode 2: A handed over as Aᵀ (k×m) — the M-contiguous operand path of the FP32 projection."""
    g = torch.Generator(device="cuda").manual_seed(m + 5 * n + 11 * k)
    at = torch.randn(k, m, device="cuda", generator=g)
    b = torch.randn(n, k, device="cuda", generator=g)
    c = torch.full((m, n), float("nan"), device="cuda", dtype=torch.float64)
    lib = ours._native.load_library()
    ours._native.check(lib.psd_gemm_tf32x3(2, ours._native.ptr(at), at.stride(0), ours._native.ptr(b),
                                           b.stride(0), m, n, k, ours._native.ptr(c), c.stride(0),
                                           ours._native.stream_handle(at.device)))
    ref = at.double().T @ b.double().T
    err = ((c - ref).norm() / ref.norm()).item()
    assert err <= 2e-7 * max(1.0, np.sqrt(k)), err


@pytest.mark.parametrize("n,k", [(1, 1), (129, 5), (512, 40), (1000, 64), (777, 256)])
def test_tf32x3_mirrored_store(ours, n, k):
    g = torch.Generator(device="cuda").manual_seed(n + k)
    a = torch.randn(n, k, device="cuda", generator=g)
    b = torch.randn(n, k, device="cuda", generator=g)
    c = torch.full((n, n), float("nan"), device="cuda", dtype=torch.float32)
    _gemm(ours, 1, a, b, c)
    ref = a.double() @ b.double().T
    low = torch.tril(ref)
    ref_m = low + low.T - torch.diag(torch.diag(ref))
    assert torch.equal(c, c.T)                        # bitwise symmetric (one value per pair)
    assert ((c.double() - ref_m).norm() / ref_m.norm()).item() <= 2e-7 * np.sqrt(k) + 1e-7


def _f32_case(x, om):
    x32 = np.asarray(x, dtype=np.float32)
    om32 = np.asarray(om, dtype=np.float32)
    return x32, om32, x32.astype(np.float64), om32.astype(np.float64)


@pytest.mark.parametrize("name", [n for n in gio.names() if "w" in np.load(f"{gio.GOLDEN}/{n}.npz").files
                                  and not n.startswith(("project_", "config1_project"))])
def test_fp32_golden_inputs(ours, name):
    d = gio.load(name)
    k, l, q, alpha = int(d["k"]), int(d["l"]), int(d["q"]), float(d["alpha"])
    x32, om32, x64, om64 = _f32_case(d["x"], d["omega"])
    params = ours.RangeParams(k=k, l=l, q=q)

    def run_ours():
        if alpha > 0:
            return ours.ran_proj_scal(x32, params, alpha, None, omega=om32, dtype="fp32",
                                      return_factors=True)
        return ours.ran_proj(x32, params, None, omega=om32, dtype="fp32", return_factors=True)

    try:
        ref = (orc.ran_proj_scal(x64, k, l, q, alpha, omega=om64) if alpha > 0
               else orc.ran_proj(x64, k, l, q, omega=om64))
    except orc.OracleError as e:  # e.g. fp32 rounding pushed the asymmetry past the tolerance
        with pytest.raises(ours.errors.REGISTRY[e.kind]):
            run_ours()
        return
    rep = run_ours()
    assert rep.result.dtype == np.float32
    np.testing.assert_array_equal(rep.result, rep.result.T)
    # eigenvalues of T within fp32 noise of the clipping threshold may land on
    # either side of it: the rank must lie between the unambiguous counts
    if ref.eigenvalues is None:
        assert rep.effective_rank == ref.effective_rank
    else:
        ev = np.asarray(ref.eigenvalues) - (1.0 if alpha > 0 else 0.0)
        tol = 1e-5 * max(1.0, float(np.abs(np.asarray(ref.eigenvalues)).max(initial=0.0)))
        assert int((ev > tol).sum()) <= rep.effective_rank <= int((ev > -tol).sum())
    assert _rel(rep.result, ref.result) <= TOL32, _rel(rep.result, ref.result)


@pytest.mark.parametrize("n", [2048, 4096])
def test_fp32_config3_shape(ours, n):
    """C3 spectrum at reduced n, k=256, p=16, q=1 (κ(Y)≈1e8 unstabilised: the
    FP32 path must re-orthonormalise — SURVEY Appendix A3)."""
    x = orc.c3_matrix(n, seed=11)
    om = np.random.default_rng(12).standard_normal((n, 272))
    x32, om32, x64, om64 = _f32_case(x, om)
    ref = orc.ran_proj(x64, 256, 16, 1, omega=om64)
    rep = ours.ran_proj(x32, ours.RangeParams(k=256, l=16, q=1), None, omega=om32, dtype="fp32")
    assert rep.effective_rank == ref.effective_rank
    assert _rel(rep.result, ref.result) <= TOL32, _rel(rep.result, ref.result)


def test_fp32_config2_shape(ours):
    """Wigner (flat spectrum: the hard case for 1xTF32), k=128, p=16, q=2."""
    n = 4096
    x = orc.wigner(n, seed=5)
    om = np.random.default_rng(6).standard_normal((n, 144))
    x32, om32, x64, om64 = _f32_case(x, om)
    ref = orc.ran_proj(x64, 128, 16, 2, omega=om64)
    rep = ours.ran_proj(x32, ours.RangeParams(k=128, l=16, q=2), None, omega=om32, dtype="fp32")
    assert rep.effective_rank == ref.effective_rank
    assert _rel(rep.result, ref.result) <= TOL32, _rel(rep.result, ref.result)


def test_fp32_torch_device_roundtrip(ours):
    n = 700
    x = torch.from_numpy(orc.wigner(n, seed=9)).float().cuda()
    x = (x + x.T) / 2
    rep = ours.ran_proj(x, ours.RangeParams(k=20, l=5, q=1), 3, dtype="fp32")
    assert isinstance(rep.result, torch.Tensor) and rep.result.is_cuda
    assert rep.result.dtype == torch.float32
    assert torch.equal(rep.result, rep.result.T)


def test_fp32_errors(ours):
    x = np.random.default_rng(0).standard_normal((64, 64)).astype(np.float32)
    with pytest.raises(ours.errors.REGISTRY["AsymmetricMatrixError"]):
        ours.ran_proj(x, ours.RangeParams(k=4, l=2), 0, dtype="fp32")
    s = (x + x.T) / 2
    with pytest.raises(ours.errors.REGISTRY["InvalidParams"]):
        ours.ran_proj(s, ours.RangeParams(k=60, l=10), 0, dtype="fp32")
    with pytest.raises(ours.errors.REGISTRY["AlphaTooSmall"]):
        ours.ran_proj_scal(s, ours.RangeParams(k=4, l=2), 1e-30, 0, dtype="fp32")


def test_fp32_project_dispatch(ours):
    n = 300
    x = orc.c1_matrix(seed=4, n=n)
    cfg = ours.ProjectorConfig(method="scaled_randomized", params=ours.RangeParams(k=20, l=10, q=2),
                               power_N=10, dtype="fp32")
    rep = ours.project(x, cfg, 5)
    ref = orc.project_scaled(np.float32(x).astype(np.float64), 20, 10, 2, power_n=10,
                             rng=np.random.default_rng(5))
    assert rep.result.dtype == np.float32
    assert _rel(rep.result, ref.result) <= TOL32


def test_fp32_full_config3_vs_fp64_path(ours):
    """Full BASELINE config-3 size (n=32768, k=256, p=16, q=1): the FP32 path
    against the FP64 path (itself pinned to the oracle at 1e-10) on the same
    fp32-rounded X and Ω — the size-independent form of the 1e-4 bar."""
    n = 32768
    x64 = ours.workloads.c3_device(n, seed=3, device="cuda")
    x32 = x64.float()
    x64.copy_(x32)
    g = torch.Generator(device="cuda").manual_seed(5)
    om = torch.randn(n, 272, device="cuda", dtype=torch.float64, generator=g).float().double()
    params = ours.RangeParams(k=256, l=16, q=1)
    r64 = ours.ran_proj(x64, params, None, omega=om).result
    del x64
    rep = ours.ran_proj(x32, params, None, omega=om, dtype="fp32")
    err = ((rep.result.double() - r64).norm() / r64.norm()).item()
    assert err <= TOL32, err
    assert torch.equal(rep.result, rep.result.T)
