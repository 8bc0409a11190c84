"""Pipelined batches (psd_plan_prefetch / ``ran_proj(..., prefetch=next_x)``): the
next matrix's require_symmetric pass and INT8 residue planes run on a side stream
during the current projection.  Every result must be BITWISE identical to the
unpipelined call on the same X and Ω (the same kernels produce the same planes),
a mismatched hint must be harmless, and the prefetched symmetry verdict must
raise exactly as the in-call one does (symmetric.py:39-57 via projection.py:100)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N = 3584          # ≥ 3072: the INT8 engine (the only one that prefetches)
K, L, Q = 48, 8, 1


@pytest.fixture(scope="module")
def psd():
    import paper_2410_19208_b200 as m
    m._native.load_library()
    return m


def _mats(count, seed=0):
    out = []
    for s in range(count):
        g = torch.Generator(device="cuda").manual_seed(100 + seed + s)
        a = torch.randn((N, N), dtype=torch.float64, device="cuda", generator=g)
        u = torch.linalg.qr(torch.randn((N, 40), dtype=torch.float64, device="cuda", generator=g))[0]
        x = (a + a.T) * (0.5 / N ** 0.5) + u @ torch.diag(torch.logspace(2, 0, 40, dtype=torch.float64,
                                                                          device="cuda")) @ u.T
        out.append(((x + x.T) / 2).contiguous())
    return out


def _omegas(count):
    g = torch.Generator(device="cuda").manual_seed(7)
    return [torch.randn((N, K + L), dtype=torch.float64, device="cuda", generator=g) for _ in range(count)]


def test_prefetched_results_are_bitwise_identical(psd):
    xs, oms = _mats(4), _omegas(4)
    params = psd.RangeParams(k=K, l=L, q=Q)
    base = [psd.ran_proj(x, params, None, omega=o, return_factors=True) for x, o in zip(xs, oms)]
    piped = []
    for i, (x, o) in enumerate(zip(xs, oms)):
        nxt = xs[i + 1] if i + 1 < len(xs) else None
        piped.append(psd.ran_proj(x, params, None, omega=o, return_factors=True, prefetch=nxt))
    torch.cuda.synchronize()
    for b, p in zip(base, piped):
        assert p.device_info["sketch_engine"] == 1
        assert p.effective_rank == b.effective_rank and p.basis_width == b.basis_width
        assert torch.equal(p.result, b.result)
        assert torch.equal(p.factors[0], b.factors[0]) and torch.equal(p.factors[1], b.factors[1])


def test_mismatched_hint_is_dropped(psd):
    xs, oms = _mats(3, seed=10), _omegas(3)
    params = psd.RangeParams(k=K, l=L, q=Q)
    ref = psd.ran_proj(xs[2], params, None, omega=oms[2])
    # hint X1, then project X2: the prefetch of X1 is discarded, X2 validated in the call
    psd.ran_proj(xs[0], params, None, omega=oms[0], prefetch=xs[1])
    got = psd.ran_proj(xs[2], params, None, omega=oms[2])
    assert torch.equal(got.result, ref.result)
    # the hint survives an FP32 call in between only as "ignored": the FP64 call after it
    # still matches
    psd.ran_proj(xs[0], params, None, omega=oms[0], prefetch=xs[1])
    psd.ran_proj(xs[0].float(), params, None, omega=oms[0].float(), dtype="fp32")
    got = psd.ran_proj(xs[2], params, None, omega=oms[2])
    assert torch.equal(got.result, ref.result)


def test_prefetched_verdict_raises_for_asymmetric_x(psd):
    xs, oms = _mats(2, seed=20), _omegas(2)
    bad = xs[1].clone()
    bad[5, 9] += 1e-3 * bad.abs().max()            # far beyond 1e-10·max|x|
    params = psd.RangeParams(k=K, l=L, q=Q)
    psd.ran_proj(xs[0], params, None, omega=oms[0], prefetch=bad)
    with pytest.raises(psd.AsymmetricMatrixError):
        psd.ran_proj(bad, params, None, omega=oms[1])
    # and the plan keeps working afterwards
    ok = psd.ran_proj(xs[0], params, None, omega=oms[0])
    assert torch.isfinite(ok.result).all()


def test_prefetched_verdict_flags_non_finite(psd):
    xs, oms = _mats(2, seed=30), _omegas(2)
    bad = xs[1].clone()
    bad[3, 3] = float("nan")
    params = psd.RangeParams(k=K, l=L, q=Q)
    psd.ran_proj(xs[0], params, None, omega=oms[0], prefetch=bad)
    with pytest.raises(psd.ConvergenceFailure):
        psd.ran_proj(bad, params, None, omega=oms[1])


def test_non_bitwise_symmetric_prefetch_uses_transpose_branch(psd):
    # within tolerance but not bitwise symmetric: the prefetched verdict must route Xᵀ·P to
    # the transposed kernel exactly as the in-call verdict does
    xs, oms = _mats(2, seed=40), _omegas(2)
    nb = xs[1].clone()
    nb[7, 2] = np.nextafter(nb[7, 2].item(), np.inf)
    params = psd.RangeParams(k=K, l=L, q=Q)
    ref = psd.ran_proj(nb, params, None, omega=oms[1])
    psd.ran_proj(xs[0], params, None, omega=oms[0], prefetch=nb)
    got = psd.ran_proj(nb, params, None, omega=oms[1])
    assert ref.device_info["used_transpose"] == 1 and got.device_info["used_transpose"] == 1
    assert torch.equal(got.result, ref.result)


def test_first_call_of_a_fresh_plan_can_be_hinted(psd):
    # a hinted call runs on the plan's non-blocking high-priority stream; buffers the plan
    # allocates lazily (and zeroes on the legacy stream) must be ready before it writes them
    psd._native.free_plans()
    torch.cuda.empty_cache()
    xs, oms = _mats(3, seed=50), _omegas(3)
    params = psd.RangeParams(k=K, l=L, q=Q)
    piped = [psd.ran_proj(x, params, None, omega=o, prefetch=xs[i + 1] if i < 2 else None)
             for i, (x, o) in enumerate(zip(xs, oms))]
    psd._native.free_plans()
    base = [psd.ran_proj(x, params, None, omega=o) for x, o in zip(xs, oms)]
    for b, p in zip(base, piped):
        assert torch.equal(p.result, b.result)


def test_fp32_prefetch_bitwise_identical(psd):
    xs, oms = _mats(3, seed=60), _omegas(3)
    xs = [x.float().contiguous() for x in xs]
    oms = [o.float() for o in oms]
    params = psd.RangeParams(k=K, l=L, q=Q)
    base = [psd.ran_proj(x, params, None, omega=o, dtype="fp32").result for x, o in zip(xs, oms)]
    piped = [psd.ran_proj(x, params, None, omega=o, dtype="fp32", prefetch=xs[i + 1] if i < 2 else None).result
             for i, (x, o) in enumerate(zip(xs, oms))]
    for b, p in zip(base, piped):
        assert p.dtype == torch.float32 and torch.equal(p, b)


def test_fp32_prefetched_verdict_raises(psd):
    xs, oms = _mats(2, seed=70), _omegas(2)
    xs = [x.float().contiguous() for x in xs]
    bad = xs[1].clone()
    bad[4, 11] += 1e-2 * bad.abs().max()
    params = psd.RangeParams(k=K, l=L, q=Q)
    psd.ran_proj(xs[0], params, None, omega=oms[0].float(), dtype="fp32", prefetch=bad)
    with pytest.raises(psd.AsymmetricMatrixError):
        psd.ran_proj(bad, params, None, omega=oms[1].float(), dtype="fp32")
