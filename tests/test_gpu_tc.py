"""Parity of the tensor-core vote path (K3-TC, tcgen05 fp16-split MMA) against the oracle.

K3-TC evaluates the bound levels; its counts are bounds, so the bar is the one of
RV_MODE_BOUND at its own threshold t' = cos(min(pi, eps + r(c))) - guard - 1.5e-5: every pair
more than 1e-5 from t' is decided as the oracle decides it.  The raw scores are also checked
against the oracle's exact s - t' (error far below the guard), and whole solves with the
tensor path enabled must return the oracle's (cell, votes) and rotation."""
import math

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu
GUARD_TC = 1e-5 + 1.5e-5
BAND = 1e-5


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def rvtc(torch_cuda):
    from paper_2506_11547_b200 import RotVote, build
    build.build()
    oracle.build()
    ctx = RotVote(max_n=4096 * 1000 + 4096, max_problems=4096, tensor_vote=True)
    yield ctx
    ctx.close()


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def test_tc_scores_match_oracle(rvtc, torch_cuda):
    torch = torch_cuda
    rng = np.random.default_rng(0)
    worst = 0.0
    for n, eps in ((3000, 0.05), (257, 0.9), (20001, 0.08)):
        pr = datagen.make_problem(n, n // 10, 0.01, eps, seed=n)
        x, y = dev(torch, pr.x), dev(torch, pr.y)
        for B in (15, 45, 360):
            lins = np.sort(rng.choice(oracle.candidates(B), 200, replace=False)).astype(np.uint32)
            sc = rvtc.debug_tc_scores(x, y, B, lins, eps)
            assert sc.shape[1] == (n + 255) // 256 * 256
            assert np.all(sc[:, n:] == -1.0)
            for c in range(0, 200, 13):
                q = oracle.cell_quat(B, int(lins[c]))
                s = oracle.pair_stats(pr.x, pr.y, q)
                t = oracle.cell_bound_threshold(B, int(lins[c]), eps) - GUARD_TC
                worst = max(worst, float(np.abs(sc[c, :n] - (s - t)).max()))
    assert worst < 2e-6, worst      # measured ~4e-7; the guard assumes <= 1.3e-5


@pytest.mark.parametrize("n", [100, 10000, 70001])
def test_tc_bound_counts_parity(rvtc, torch_cuda, n):
    from paper_2506_11547_b200 import RV_MODE_BOUND_TC
    torch = torch_cuda
    pr = datagen.make_problem(n, n // 10, 0.01, 0.05, seed=7)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    rng = np.random.default_rng(1)
    for B in (5, 15, 45, 90):
        cand = oracle.candidates(B)
        lins = np.sort(rng.choice(cand, min(cand.size, 1500), replace=False)).astype(np.uint32)
        got = rvtc.count_cells(x, y, B, lins, pr.eps, RV_MODE_BOUND_TC)
        thr = np.array([oracle.cell_bound_threshold(B, int(l), pr.eps) for l in lins]) - GUARD_TC
        lo, _ = oracle.count_cells(pr.x, pr.y, B, lins, thr + BAND, band=0)
        hi, _ = oracle.count_cells(pr.x, pr.y, B, lins, thr - BAND, band=0)
        assert np.all(got >= lo) and np.all(got <= hi), B


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_tc_solve_matches_oracle(rvtc, torch_cuda, cfg):
    torch = torch_cuda
    pr = datagen.CONFIGS[cfg]()
    ref = oracle.solve(pr.x, pr.y, pr.eps)
    res = rvtc.solve(dev(torch, pr.x), dev(torch, pr.y), pr.eps)
    assert (res.cell, res.votes, res.n_tied) == (ref.cell, ref.votes, ref.n_tied)
    assert oracle.rotation_angle_between(res.q, ref.q) < 1e-9
    for L in (2, 3, 6):
        r = rvtc.solve(dev(torch, pr.x), dev(torch, pr.y), pr.eps, levels=L)
        assert (r.cell, r.votes, r.n_tied) == (ref.cell, ref.votes, ref.n_tied)


def test_tc_batched_matches_oracle(rvtc, torch_cuda):
    torch = torch_cuda
    rng = np.random.default_rng(5)
    probs = [datagen.make_problem(int(rng.integers(2, 2000)), 60, float(rng.uniform(.005, .03)),
                                  0.09, seed=[5, p]) for p in range(24)]
    bt = datagen.batch_of(probs, 0.09)
    res = rvtc.solve_batched(dev(torch, bt.x), dev(torch, bt.y), bt.offsets, bt.eps)
    for p, r in zip(probs, res):
        ref = oracle.solve(p.x, p.y, bt.eps)
        assert (r.cell, r.votes, r.n_tied) == (ref.cell, ref.votes, ref.n_tied)
        assert oracle.rotation_angle_between(r.q, ref.q) < 1e-9


def test_tc_fullsize_cfg4(rvtc, torch_cuda):
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    pr = datagen.cfg4()
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    a = rvtc.solve(x, y, pr.eps)
    f = RotVote(max_n=pr.n, tensor_vote=False)
    b = f.solve(x, y, pr.eps)
    f.close()
    assert (a.cell, a.votes, a.n_tied) == (b.cell, b.votes, b.n_tied)
    assert np.array_equal(a.q, b.q)
    cnt, nr = oracle.count_cells(pr.x, pr.y, 360, [a.lin], math.cos(pr.eps), band=1e-12)
    assert a.votes == cnt[0]


@pytest.mark.parametrize("n", [100, 10000, 70001])
def test_tc_final_counts_parity(rvtc, torch_cuda, n):
    """RV_MODE_FINAL_TC: two thresholds per cell (two TMEM lanes); cnt_b <= exact <= cnt_a."""
    from paper_2506_11547_b200 import RV_MODE_FINAL_TC
    torch = torch_cuda
    pr = datagen.make_problem(n, n // 10, 0.01, 0.05, seed=8)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    rng = np.random.default_rng(2)
    tau = math.cos(pr.eps)
    ref = oracle.solve(pr.x, pr.y, pr.eps)
    i, j, k = ref.cell
    near = [oracle.lin_of(360, i + a, j + b, k + c) for a in (-1, 0, 1) for b in (-1, 0, 1)
            for c in (-1, 0, 1)]
    lins = np.unique(np.concatenate([rng.choice(oracle.candidates(360), 300, replace=False),
                                     near]).astype(np.uint32))
    a, b = rvtc.count_cells(x, y, 360, lins, pr.eps, RV_MODE_FINAL_TC)
    for cnt, thr in ((a, tau - GUARD_TC), (b, tau + GUARD_TC)):
        lo, _ = oracle.count_cells(pr.x, pr.y, 360, lins, thr + BAND, band=0)
        hi, _ = oracle.count_cells(pr.x, pr.y, 360, lins, thr - BAND, band=0)
        assert np.all(cnt >= lo) and np.all(cnt <= hi)
    exact, _ = oracle.count_cells(pr.x, pr.y, 360, lins, tau, band=0)
    assert np.all(b <= exact) and np.all(exact <= a)


def test_tc_loopback_and_nccl_paths(torch_cuda):
    """The sharded paths (loopback ranks, 1-rank NCCL communicator) with the tensor-core
    vote give the one-rank answer, on both culled vote paths (K3-CT, the default, and the FP32
    K3-C): the same (cell, votes, ties, q) and the same searched pairs (pair_votes)."""
    from paper_2506_11547_b200 import RotVote, rot_vote_get_unique_id
    torch = torch_cuda
    pr = datagen.cfg2(seed=9)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    answers = []
    for path in ("tc", "fp32"):
        base = RotVote(max_n=1 << 16, cull=path)
        ref = base.solve(x, y, pr.eps)
        base.close()
        for kw in (dict(emulate_world=3), dict(nccl_id=rot_vote_get_unique_id())):
            ctx = RotVote(max_n=1 << 16, cull=path, **kw)
            r = ctx.solve(x, y, pr.eps)
            ctx.close()
            assert (r.cell, r.votes, r.n_tied, r.pair_votes) == (ref.cell, ref.votes, ref.n_tied,
                                                                 ref.pair_votes), (path, kw)
            assert np.array_equal(r.q, ref.q)
        answers.append(ref)
    assert (answers[0].cell, answers[0].votes, answers[0].n_tied) == \
        (answers[1].cell, answers[1].votes, answers[1].n_tied)
    assert np.array_equal(answers[0].q, answers[1].q)
