"""ran_proj_many: host matrices streamed through the GPU with the uploads and
downloads overlapped — per-matrix results identical to one ran_proj /
ran_proj_scal call each with the same Ω stream."""

import numpy as np
import pytest
import torch


@pytest.fixture(scope="module")
def psd():
    import paper_2410_19208_b200 as m
    return m


def _sym(n, seed):
    x = np.random.default_rng(seed).standard_normal((n, n))
    return (x + x.T) / 2


def test_rejects_non_square_before_touching_the_gpu(psd):
    with pytest.raises(psd.NonSquareError):
        psd.ran_proj_many([np.zeros((3, 4))], psd.RangeParams(k=1, l=1), rng=0)
    assert psd.ran_proj_many([], psd.RangeParams(k=1, l=1), rng=0) == []


@pytest.mark.gpu
@pytest.mark.parametrize("alpha", [None, 0.5])
def test_matches_sequential_calls_numpy(psd, alpha):
    xs = [_sym(300, s) for s in range(5)]
    params = psd.RangeParams(k=20, l=6, q=1)
    reps = psd.ran_proj_many(xs, params, np.random.default_rng(9), alpha=alpha)
    rng = np.random.default_rng(9)
    for x, rep in zip(xs, reps):
        ref = psd.ran_proj(x, params, rng) if alpha is None else psd.ran_proj_scal(x, params, alpha, rng)
        assert isinstance(rep.result, np.ndarray)
        np.testing.assert_array_equal(rep.result, ref.result)
        assert rep.effective_rank == ref.effective_rank


@pytest.mark.gpu
def test_pinned_torch_inputs_and_outputs(psd):
    xs = [torch.from_numpy(_sym(256, 10 + s)).pin_memory() for s in range(3)]
    outs = [torch.empty((256, 256), dtype=torch.float64).pin_memory() for _ in xs]
    params = psd.RangeParams(k=16, l=8, q=2)
    reps = psd.ran_proj_many(xs, params, np.random.default_rng(4), out=outs)
    rng = np.random.default_rng(4)
    for x, o, rep in zip(xs, outs, reps):
        assert rep.result is o
        ref = psd.ran_proj(x.numpy(), params, rng).result
        np.testing.assert_array_equal(o.numpy(), ref)


@pytest.mark.gpu
def test_rejects_device_inputs(psd):
    with pytest.raises(psd.InvalidParams):
        psd.ran_proj_many([torch.zeros((8, 8), dtype=torch.float64, device="cuda")],
                          psd.RangeParams(k=2, l=2), rng=0)


@pytest.mark.gpu
def test_ran_proj_out_buffer(psd):
    x = torch.from_numpy(_sym(200, 3)).cuda()
    params = psd.RangeParams(k=12, l=6, q=1)
    buf = torch.empty((200, 200), dtype=torch.float64, device="cuda")
    rep = psd.ran_proj(x, params, np.random.default_rng(1), out=buf)
    assert rep.result.data_ptr() == buf.data_ptr()
    ref = psd.ran_proj(x, params, np.random.default_rng(1))
    assert torch.equal(buf, ref.result)
    with pytest.raises(psd.InvalidParams):
        psd.ran_proj(x, params, np.random.default_rng(1), out=torch.empty((200, 199), dtype=torch.float64,
                                                                             device="cuda"))
