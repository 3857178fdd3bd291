"""The device-resident level loop of batched solves (csrc/rv_dplan.cu) against the host
planner (rv_plan.cpp, forced with planner="host") and the oracle.

The device loop takes the planner's decisions on the GPU; it must return the same winner,
votes, ties, lb* and recheck sets as the host planner on every problem, for several chains
and `levels`, ragged sizes (n = 2 ... 3000), both vote paths (FP32 and tensor core), and its
per-phase block counts must be the host planner's (dive picks compare excess values computed
with the device's cos(); a last-ulp difference could only reorder an exact tie, so a tiny
fraction of mismatching phase lists is tolerated and reported)."""
import os

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


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def host_plan(ctx, fn):
    """fn run on a twin of ctx whose levels are driven by the host planner (planner="host")."""
    h = ctx.twin(planner="host")
    try:
        return fn(h)
    finally:
        h.close()


def compare(res_d, res_h, strict_phases=False):
    mism = 0
    for p, (a, b) in enumerate(zip(res_d, res_h)):
        assert (a.cell, a.votes, a.n_tied) == (b.cell, b.votes, b.n_tied), p
        assert np.array_equal(a.q, b.q), p
        assert (a.n_inliers, a.flags) == (b.n_inliers, b.flags), p
        if a.cells_per_phase != b.cells_per_phase:
            mism += 1
        else:
            assert (a.lb_star, a.n_rechecked, a.cells_evaluated, a.pair_votes) == \
                   (b.lb_star, b.n_rechecked, b.cells_evaluated, b.pair_votes), p
    if strict_phases:
        assert mism == 0
    assert mism <= max(1, len(res_d) // 500), mism
    return mism


def ragged_batch(seed, P, nmax, eps):
    rng = np.random.default_rng(seed)
    probs = []
    for p in range(P):
        n = int(rng.integers(2, nmax))
        probs.append(datagen.make_problem(n, int(rng.integers(0, n + 1)),
                                          float(rng.uniform(0.0, 0.03)), eps, seed=[seed, p]))
    return datagen.batch_of(probs, eps)


@pytest.mark.parametrize("tensor_vote", [False, True])
@pytest.mark.parametrize("chain,levels", [(None, 0), ((5, 15, 45), 2), ((15, 45, 90, 180), 3), ((4, 8, 16, 32), 4),
                                          ((3, 9, 27, 81), 3), ((6, 18, 90), 3)])
def test_device_loop_equals_host_planner(torch_cuda, tensor_vote, chain, levels):
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    bt = ragged_batch(5 + levels, 96, 3000, 0.1)
    ctx = RotVote(max_n=int(bt.offsets[-1]) + 16, max_problems=96, chain=chain, cull=False,
                  tensor_vote=tensor_vote)
    try:
        x, y = dev(torch, bt.x), dev(torch, bt.y)
        rd = ctx.solve_batched(x, y, bt.offsets, bt.eps, levels=levels)
        rh = host_plan(ctx, lambda c: c.solve_batched(x, y, bt.offsets, bt.eps, levels=levels))
        compare(rd, rh)
        # and the oracle (certified == exhaustive) on a sample
        for p in range(0, 96, 17):
            pr = bt.problems[p]
            ref = oracle.solve(pr.x, pr.y, bt.eps, chain=ctx.chain,
                               levels=levels if levels else min(5, len(ctx.chain)))
            assert (rd[p].votes, rd[p].n_tied) == (ref.votes, ref.n_tied), p
    finally:
        ctx.close()


def test_device_loop_cfg5_equals_host_planner(torch_cuda):
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    bt = datagen.cfg5()
    ctx = RotVote(max_n=int(bt.offsets[-1]) + 16, max_problems=4096, tensor_vote=True, cull=False)
    try:
        x, y = dev(torch, bt.x), dev(torch, bt.y)
        rd = ctx.solve_batched(x, y, bt.offsets, bt.eps)
        rh = host_plan(ctx, lambda c: c.solve_batched(x, y, bt.offsets, bt.eps))
        mism = compare(rd, rh)
        print("cfg5 phase-list mismatches:", mism)
        # repeated calls reuse the context's buffers and give identical answers
        rd2 = ctx.solve_batched(x, y, bt.offsets, bt.eps)
        for a, b in zip(rd, rd2):
            assert (a.cell, a.votes, a.cells_per_phase) == (b.cell, b.votes, b.cells_per_phase)
    finally:
        ctx.close()


def test_device_loop_degenerate_batches(torch_cuda):
    """n = 2 problems, all-outlier problems, exact antipodal pairs (y = -x), one problem."""
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    probs = [datagen.make_problem(2, 2, 0.0, 0.2, seed=1),
             datagen.make_problem(2, 0, 0.0, 0.2, seed=2),
             datagen.make_problem(50, 0, 0.0, 0.2, seed=3),
             datagen.make_problem(300, 300, 0.0, 0.2, seed=4)]
    anti = datagen.make_problem(40, 0, 0.0, 0.2, seed=5)
    anti.y[:] = -anti.x
    probs.append(anti)
    bt = datagen.batch_of(probs, 0.2)
    ctx = RotVote(max_n=4096, max_problems=8, cull=False)
    try:
        x, y = dev(torch, bt.x), dev(torch, bt.y)
        rd = ctx.solve_batched(x, y, bt.offsets, bt.eps)
        rh = host_plan(ctx, lambda c: c.solve_batched(x, y, bt.offsets, bt.eps))
        compare(rd, rh, strict_phases=True)
        for pr, r in zip(probs, rd):
            ref = oracle.solve(pr.x, pr.y, bt.eps)
            assert (r.votes, r.n_tied) == (ref.votes, ref.n_tied)
        one = datagen.batch_of(probs[3:4], 0.2)
        r1 = ctx.solve_batched(dev(torch, one.x), dev(torch, one.y), one.offsets, one.eps)
        assert (r1[0].cell, r1[0].votes) == (rd[3].cell, rd[3].votes)
    finally:
        ctx.close()


def test_device_loop_large_single_problems(torch_cuda):
    """One-problem batches of 2e4 ... 1e6 correspondences (many correspondence chunks per
    item, uneven last chunks) through the device loop equal the host-planner solve."""
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    ctx = RotVote(max_n=1_000_000, cull=False)
    try:
        cases = [datagen.make_problem(20_000, 400, 0.01, 0.05, seed=81),
                 datagen.make_problem(70_001, 700, 0.01, 0.05, seed=82),
                 datagen.make_problem(250_000, 2_500, 0.01, 0.05, seed=83),
                 datagen.cfg4()]
        for pr in cases:
            x, y = dev(torch, pr.x), dev(torch, pr.y)
            rb = ctx.solve_batched(x, y, np.array([0, pr.n], np.int64), pr.eps)
            rs = host_plan(ctx, lambda c: c.solve(x, y, pr.eps))
            compare(rb, [rs], strict_phases=True)
    finally:
        ctx.close()


@pytest.mark.parametrize("tensor_vote", [False, True])
def test_single_solve_device_loop_equals_host_planner(torch_cuda, tensor_vote):
    """rot_vote_solve on one GPU takes the device loop (P = 1); the host planner (the
    sharding path, planner="host") must agree on every field, incl. per-phase block counts."""
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    ctx = RotVote(max_n=200_000, tensor_vote=tensor_vote, cull=False)
    try:
        cases = [datagen.cfg1(), datagen.cfg2(seed=3), datagen.cfg3(seed=4)]
        rng = np.random.default_rng(77)
        for k in range(6):
            n = int(rng.integers(2, 20_000))
            cases.append(datagen.make_problem(n, int(rng.integers(0, n + 1)), 0.01, 0.05,
                                              seed=[77, k]))
        for pr in cases:
            x, y = dev(torch, pr.x), dev(torch, pr.y)
            for levels in (0, 2, 3):
                rd = ctx.solve(x, y, pr.eps, levels=levels)
                rh = host_plan(ctx, lambda c: c.solve(x, y, pr.eps, levels=levels))
                compare([rd], [rh], strict_phases=True)
    finally:
        ctx.close()


@pytest.mark.parametrize("tensor_vote", [False, True])
def test_sharded_single_solve_loopback(torch_cuda, tensor_vote):
    """One problem over W emulated ranks (emulate_world): every level's list is built in
    parent order and its votes are split into W slices -- the code path of the NCCL run with
    the all-gather replaced by in-place writes.  Every field must equal the one-rank solve, and
    the host planner's sharded path (planner="host")."""
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    cases = [datagen.cfg2(seed=5), datagen.cfg3(seed=6),
             datagen.make_problem(3, 2, 0.0, 0.1, seed=7),
             datagen.make_problem(40_000, 400, 0.01, 0.05, seed=8)]
    for pr in cases:
        x, y = dev(torch, pr.x), dev(torch, pr.y)
        ref = None
        for W in (1, 2, 3, 4, 8):
            ctx = RotVote(max_n=1 << 17, emulate_world=W, tensor_vote=tensor_vote, cull=False)
            try:
                r = ctx.solve(x, y, pr.eps)
                rh = host_plan(ctx, lambda c: c.solve(x, y, pr.eps))
            finally:
                ctx.close()
            compare([r], [rh], strict_phases=True)
            if ref is None:
                ref = r
            else:
                compare([r], [ref], strict_phases=True)
