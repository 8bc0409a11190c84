"""Reconstruction X̂₊ = W·diag(d)·Wᵀ (projection.py:72-78) on the INT8 tensor
cores (Ozaki scheme I digit slices, csrc/ozaki_syrk.cu) — the default
reconstruction of the FP64 projection whenever its products run on the INT8
engine (n >= 3072).

V = W·diag(√d); row i is truncated to a 49-bit integer relative to 2^e_i
(max_k |v_ik| < 2^e_i) and split into 7 base-128 int8 digits; the digit
products of level t+u <= 6 are summed exactly.  Per entry the truncation costs
<= 2·r·2^(e_i+e_j−49) and the dropped levels <= 6.1·r·2^(e_i+e_j−49), so
|X̂ − VVᵀ|_ij <= 2^-45·r·2^(e_i+e_j) <= 2^-43·r·max|v_i|·max|v_j| — the test
bound below, plus FP64 rounding of the torch reference itself.
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

int8_enabled = pytest.mark.skipif(os.environ.get("PSD_FP64_OZAKI", "") == "0",
                                  reason="INT8 engine disabled by PSD_FP64_OZAKI=0")
syrk_enabled = pytest.mark.skipif(os.environ.get("PSD_OZ_SYRK", "") == "0",
                                  reason="INT8 reconstruction disabled by PSD_OZ_SYRK=0")


@pytest.fixture(scope="module")
def ours():
    import paper_2410_19208_b200 as m
    m._native.load_library()
    return m


def _syrk(ours, w, d, ldr=None):
    lib = ours._native.load_library()
    n, r = w.shape
    ldr = ldr or n
    buf = torch.full((n, ldr), float("nan"), dtype=torch.float64, device=w.device)
    ours._native.check(lib.psd_syrk_f64_int8(ours._native.ptr(w), w.stride(0), ours._native.ptr(d), n, r,
                                             ours._native.ptr(buf), ldr, ours._native.stream_handle(w.device)))
    torch.cuda.synchronize()
    return buf[:, :n]


def _check(w, d, c):
    n, r = w.shape
    ref = (w * d) @ w.T
    v = w * d.sqrt()
    rv = v.abs().amax(dim=1, keepdim=True)
    bound = r * 2.0 ** -43 * (rv @ rv.T) + 2 * r * 2.0 ** -52 * ((w.abs() * d) @ w.abs().T)
    assert torch.isfinite(c).all()
    assert torch.equal(c, c.T), "result must be bitwise symmetric"
    excess = ((c - ref).abs() - bound).max().item()
    assert excess <= 0.0, f"entry error above the bound by {excess:.3e}"
    rel = (torch.linalg.norm(c - ref) / torch.linalg.norm(ref)).item()
    return rel


@pytest.mark.parametrize("n,r", [(256, 16), (300, 40), (1000, 50), (129, 33), (1, 1), (33, 7),
                                 (2048, 158), (4096, 272), (640, 544), (777, 640),
                                 (1000, 170), (1100, 200), (900, 224), (700, 225)])
def test_syrk_matches_fp64(ours, n, r):
    g = torch.Generator(device="cpu").manual_seed(n * 31 + r)
    w = torch.linalg.qr(torch.randn(n, r, generator=g, dtype=torch.float64))[0] if n >= r else \
        torch.randn(n, r, generator=g, dtype=torch.float64)
    d = torch.rand(r, generator=g, dtype=torch.float64) * 100.0 + 1e-3
    w, d = w.cuda().contiguous(), d.cuda()
    rel = _check(w, d, _syrk(ours, w, d))
    assert rel <= 1e-13


def test_syrk_extreme_rows_and_zeros(ours):
    g = torch.Generator(device="cpu").manual_seed(7)
    n, r = 1500, 96
    w = torch.randn(n, r, generator=g, dtype=torch.float64)
    w[::7] *= 1e-9
    w[3::11] *= 1e7
    w[5] = 0.0
    w[:, 10] = 0.0
    w[40, :50] = 0.0
    d = torch.logspace(4, -6, r, dtype=torch.float64)
    w, d = w.cuda(), d.cuda()
    c = _syrk(ours, w, d)
    _check(w, d, c)
    assert (c[5] == 0).all() and (c[:, 5] == 0).all()


def test_syrk_padded_ld_and_diagonal(ours):
    g = torch.Generator(device="cpu").manual_seed(11)
    n, r = 515, 21
    wf = torch.randn(n, 40, generator=g, dtype=torch.float64).cuda()
    w = wf[:, :r]                      # ld 40 > r
    d = torch.rand(r, generator=g, dtype=torch.float64).cuda() + 0.5
    c = _syrk(ours, w, d, ldr=n + 3)   # odd ld: scalar row stores
    _check(w, d, c)
    diag = ((w * w) * d).sum(dim=1)
    assert torch.allclose(torch.diagonal(c), diag, rtol=1e-13, atol=0)


@int8_enabled
@syrk_enabled
def test_projection_uses_int8_reconstruction(ours):
    from oracle import psd_oracle as orc
    n = 3072
    x = torch.from_numpy(orc.wigner(n, seed=5)).cuda()
    om = torch.from_numpy(np.random.default_rng(6).standard_normal((n, 40))).cuda()
    rep = ours.ran_proj(x, ours.RangeParams(k=32, l=8, q=1), None, omega=om)
    assert rep.device_info["recon_engine"] == 1
    assert rep.device_info["sketch_engine"] == 1
    o = orc.ran_proj(x.cpu().numpy(), 32, 8, 1, omega=om.cpu().numpy())
    res = rep.result.cpu().numpy()
    assert np.array_equal(res, res.T)
    err = np.linalg.norm(res - o.result) / np.linalg.norm(o.result)
    assert err <= 1e-10, err


def test_syrk_rejects_wide_factor(ours):
    # the exact s32 / IMAD.WIDE level combination holds for K <= 640
    w = torch.zeros(64, 641, dtype=torch.float64, device="cuda")
    d = torch.ones(641, dtype=torch.float64, device="cuda")
    with pytest.raises(Exception):
        _syrk(ours, w, d)


@int8_enabled
@pytest.mark.parametrize("k,l,q,alpha", [(118, 20, 1, 0.0), (63, 13, 1, 0.913), (169, 25, 2, 0.429)])
def test_rank_deficient_sketch_within_reference_sensitivity(ours, k, l, q, alpha):
    """X of numerical rank 60 (+1e-4 noise), n ≥ 3072 (INT8 products and reconstruction).
    With the sketch wider than that rank at q = 1 the reference's own output moves by
    ~1e-9 under a one-ulp perturbation of X; ours must stay within 10× of that (and
    within 1e-10 whenever the problem is well conditioned).  The reference's
    sensitivity is the larger of two independent one-ulp perturbations, and ours must
    stay within 2x of it (README "Parity bar": the ill-conditioned exception)."""
    from oracle import psd_oracle as orc
    rs = np.random.default_rng(k + l + q)
    n = 3100
    u = np.linalg.qr(rs.standard_normal((n, 60)))[0]
    s = np.geomspace(1e3, 1e-2, 60) * rs.choice([-1.0, 1.0], 60)
    x = (u * s) @ u.T + 1e-4 * orc.wigner(n, seed=k)
    x = (x + x.T) / 2
    om = rs.standard_normal((n, k + l))
    run = (lambda xx: orc.ran_proj_scal(xx, k, l, q, alpha, omega=om)) if alpha > 0 else \
        (lambda xx: orc.ran_proj(xx, k, l, q, omega=om))
    ref = run(x)
    sens = 0.0
    for _ in range(2):
        e = rs.choice([-1.0, 1.0], (n, n))
        e = np.triu(e) + np.triu(e, 1).T
        sens = max(sens, np.linalg.norm(run(x * (1 + 2.0 ** -53 * e)).result - ref.result)
                   / np.linalg.norm(ref.result))
    xd, omd = torch.from_numpy(x).cuda(), torch.from_numpy(om).cuda()
    prm = ours.RangeParams(k=k, l=l, q=q)
    rep = ours.ran_proj_scal(xd, prm, alpha, None, omega=omd) if alpha > 0 else ours.ran_proj(xd, prm, None, omega=omd)
    if os.environ.get("PSD_OZ_SYRK", "") != "0":
        assert rep.device_info["recon_engine"] == 1
    assert rep.basis_width == ref.basis_width and rep.effective_rank == ref.effective_rank
    err = np.linalg.norm(rep.result.cpu().numpy() - ref.result) / np.linalg.norm(ref.result)
    assert err <= max(1e-10, 2 * sens), (err, sens)
