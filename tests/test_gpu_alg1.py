"""NEXT-4: the paper's Algorithm 1 on the GPU (csrc/rv_alg1.cu) against the oracle's
(or_alg1_bins / or_alg1_solve).  The bins are integers decided in fp64 with the same
explicitly rounded operations on both sides, so the accumulators must be identical entry by
entry, including degenerate rows (a = b, a = -b) and ragged sizes; the winner (lin, votes)
must match at full size (config 4, 1.8e8 samples)."""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def rv(torch_cuda):
    from paper_2506_11547_b200 import RotVote, build
    build.build()
    oracle.build()
    ctx = RotVote(max_n=1_000_000)
    yield ctx
    ctx.close()


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def _check_acc(torch, rv, x, y, J):
    B = 360
    acc = torch.zeros(B ** 3, dtype=torch.int32, device="cuda")
    r = rv.alg1(dev(torch, x), dev(torch, y), J=J, acc=acc)
    nz = torch.nonzero(acc).flatten()
    g_lin = nz.cpu().numpy()
    g_cnt = acc[nz].cpu().numpy()
    o_lin, o_cnt = np.unique(oracle.alg1_bins(x, y, B, J), return_counts=True)
    assert np.array_equal(g_lin, o_lin) and np.array_equal(g_cnt, o_cnt)
    # winner: max count, ties -> lowest lin
    best = o_lin[np.argmax(o_cnt)]
    assert (r["lin"], r["votes"]) == (int(best), int(o_cnt.max()))
    assert r["samples"] == x.shape[0] * J
    return r


@pytest.mark.parametrize("J", [1, 7, 180, 360])
def test_alg1_accumulator_equals_oracle(rv, torch_cuda, J):
    rng = np.random.default_rng(J)
    n = int(rng.integers(50, 3000))
    pr = datagen.make_problem(n, n // 4, 0.01, 0.05, seed=J)
    x, y = pr.x.copy(), pr.y.copy()
    y[0] = -x[0]            # antipodal (the paper leaves the axis open: reading R13)
    y[1] = x[1]             # identical vectors
    y[2] = 3.5 * x[2]       # not unit length: normalised like every row
    _check_acc(torch_cuda, rv, x, y, J)


def test_alg1_configs_1_and_2(rv, torch_cuda):
    for pr in (datagen.cfg1(), datagen.cfg2()):
        r = _check_acc(torch_cuda, rv, pr.x, pr.y, 180)
        lin, votes, q = oracle.alg1_solve(pr.x, pr.y, 360, 180)
        assert (r["lin"], r["votes"]) == (lin, votes)
        assert np.allclose(r["q"], q, atol=1e-12)


@pytest.mark.slow
def test_alg1_fullsize_cfg4(rv, torch_cuda):
    pr = datagen.cfg4()
    r = rv.alg1(dev(torch_cuda, pr.x), dev(torch_cuda, pr.y), J=180)
    lin, votes, q = oracle.alg1_solve(pr.x, pr.y, 360, 180)
    assert (r["lin"], r["votes"]) == (lin, votes)


def test_alg1_rejects_bad_rows(rv, torch_cuda):
    from paper_2506_11547_b200 import RotVoteError
    pr = datagen.make_problem(100, 10, 0.01, 0.05, seed=1)
    x = pr.x.copy()
    x[17] = 0.0
    with pytest.raises(RotVoteError):
        rv.alg1(dev(torch_cuda, x), dev(torch_cuda, pr.y), J=180)
    r = rv.alg1(dev(torch_cuda, pr.x), dev(torch_cuda, pr.y), J=180)   # context still usable
    assert r["samples"] == 100 * 180
