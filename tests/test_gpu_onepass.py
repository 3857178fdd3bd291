"""The one-pass single solve (csrc/rv_level_loop.cpp solve_one_pass: the whole certified search
and the refinement enqueued with no host round trip, one read-back per solve) against the
device loop with per-level round trips (planner="device_sync", its fallback), the host planner
(planner="host") and the oracle.

Every decision of the one-pass loop is the per-level loop's, and its fused refinement
(rv_refine1_kernel) keeps K6/K7's decomposition and summation order, so the results must be
bit-identical: winner, votes, ties, lb*, per-phase block counts, refined q, flags and the mask.
A solve that outgrows the fixed capacities or meets the re-dive trigger (R18) is redone by the
per-level loop (flag RV_RETRIED) and must still be identical."""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

RV_RETRIED = 8


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def solve_all(torch, rv, pr, levels=0):
    """(result, mask) of one solve on a context."""
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    mask = torch.zeros((pr.n + 31) // 32, dtype=torch.int32, device="cuda")
    r = rv.solve(x, y, pr.eps, levels=levels, mask=mask)
    return r, mask.cpu().numpy()


def same(a, b, ma, mb, phases=True):
    assert (a.cell, a.votes, a.n_tied, a.lb_star) == (b.cell, b.votes, b.n_tied, b.lb_star)
    assert np.array_equal(a.q, b.q), (a.q, b.q)
    assert (a.n_inliers, a.flags & ~RV_RETRIED) == (b.n_inliers, b.flags & ~RV_RETRIED)
    assert np.array_equal(ma, mb)
    if phases:
        assert a.cells_per_phase == b.cells_per_phase
        assert (a.n_rechecked, a.pair_votes) == (b.n_rechecked, b.pair_votes)


PROBLEMS = [
    ("cfg1", lambda: datagen.cfg1()),
    ("n2", lambda: datagen.make_problem(2, 2, 0.0, 0.05, seed=3)),
    ("n37", lambda: datagen.make_problem(37, 20, 0.01, 0.05, seed=4)),
    ("n4000", lambda: datagen.make_problem(4000, 400, 0.01, 0.05, seed=1)),
    ("n20k_99", lambda: datagen.make_problem(20000, 200, 0.01, 0.05, seed=2)),
    ("cfg2", lambda: datagen.cfg2()),
]


@pytest.mark.parametrize("name,mk", PROBLEMS)
@pytest.mark.parametrize("cull", [True, False])
def test_one_pass_equals_per_level_loop(torch_cuda, name, mk, cull):
    from paper_2506_11547_b200 import RotVote
    pr = mk()
    rv = RotVote(max_n=max(pr.n, 64), cull=cull)
    sync = rv.twin(planner="device_sync")
    try:
        a, ma = solve_all(torch_cuda, rv, pr)
        b, mb = solve_all(torch_cuda, sync, pr)
        same(a, b, ma, mb)
        if not a.flags & RV_RETRIED:
            assert a.host_syncs == 1, a.host_syncs
            assert b.host_syncs > a.host_syncs
            # phase times: every phase measured, their sum is the solve
            t = a.phase_ms
            assert all(v >= 0.0 for v in t.values()), t
            assert abs(sum(t.values()) - a.ms) <= 0.05 * a.ms + 0.05, (t, a.ms)
        ref = oracle.solve(pr.x, pr.y, pr.eps)
        assert (a.cell, a.votes, a.n_tied) == (ref.cell, ref.votes, ref.n_tied)
    finally:
        rv.close()
        sync.close()


@pytest.mark.parametrize("levels", [2, 3, 4, 5])
def test_one_pass_levels_and_host_planner(torch_cuda, levels):
    from paper_2506_11547_b200 import RotVote
    pr = datagen.make_problem(6000, 300, 0.01, 0.05, seed=10 + levels)
    rv = RotVote(max_n=pr.n)
    host = rv.twin(planner="host")
    try:
        a, ma = solve_all(torch_cuda, rv, pr, levels)
        b, mb = solve_all(torch_cuda, host, pr, levels)
        same(a, b, ma, mb, phases=False)
        assert a.host_syncs == 1 or a.flags & RV_RETRIED
    finally:
        rv.close()
        host.close()


def test_one_pass_retry_path(torch_cuda):
    """A wide inlier angle (eps = 0.6 rad): a correspondence passes the bound test of ~25% of
    the level-0 blocks, so the culling lists outgrow the one-pass capacity (an eighth of the
    level-0 pairs); the one-pass solve must hand the problem to the per-level loop and still
    return its exact result."""
    from paper_2506_11547_b200 import RotVote
    pr = datagen.make_problem(3000, 900, 0.01, 0.6, seed=7)
    n = pr.n
    rv = RotVote(max_n=n, chain=(15, 45, 90, 180, 360))
    sync = rv.twin(planner="device_sync")
    try:
        a, ma = solve_all(torch_cuda, rv, pr)
        b, mb = solve_all(torch_cuda, sync, pr)
        same(a, b, ma, mb)
        assert a.flags & RV_RETRIED, "expected the one-pass solve to be redone"
        assert a.host_syncs > 1
    finally:
        rv.close()
        sync.close()


def test_repeated_solves_after_a_retry(torch_cuda):
    """The same solve (same buffers: the graph key) repeated after the one-pass loop handed it to
    the per-level loop.  The retry grows capacities, so the next enqueue reallocates workspace:
    it must run directly, never as a capture (a graph captured across a reallocation keeps freed
    pointers in its earlier nodes -- an illegal access at launch, found with the rigid pose at
    99% outliers).  A growing problem size on one context walks the same reallocation path."""
    from paper_2506_11547_b200 import RotVote
    pr = datagen.make_problem(3000, 900, 0.01, 0.6, seed=7)
    rv = RotVote(max_n=40000, chain=(15, 45, 90, 180, 360))
    try:
        x, y = dev(torch_cuda, pr.x), dev(torch_cuda, pr.y)
        mask = torch_cuda.zeros((pr.n + 31) // 32, dtype=torch_cuda.int32, device="cuda")
        ref = rv.solve(x, y, pr.eps, mask=mask)
        m_ref = mask.cpu().numpy()
        assert ref.flags & RV_RETRIED
        for k in range(5):
            mask.zero_()
            r = rv.solve(x, y, pr.eps, mask=mask)
            same(r, ref, mask.cpu().numpy(), m_ref)
        # larger problems on the same context (every workspace buffer grows), each solved
        # three times: direct, capture, replay
        for n in (6000, 20000, 40000):
            pb = datagen.make_problem(n, n // 10, 0.01, 0.05, seed=n)
            xb, yb = dev(torch_cuda, pb.x), dev(torch_cuda, pb.y)
            mb = torch_cuda.zeros((n + 31) // 32, dtype=torch_cuda.int32, device="cuda")
            first = rv.solve(xb, yb, pb.eps, mask=mb)
            m_first = mb.cpu().numpy()
            for k in range(3):
                mb.zero_()
                r = rv.solve(xb, yb, pb.eps, mask=mb)
                same(r, first, mb.cpu().numpy(), m_first)
        torch_cuda.cuda.synchronize()
    finally:
        rv.close()


def test_one_pass_full_size_cfg4(torch_cuda):
    """The bench's workload (cfg4, chain 15-45-180-360): one pass, identical to the per-level
    loop, and the oracle's winner (the full oracle solve is in test_gpu_fullsize.py)."""
    from paper_2506_11547_b200 import RotVote
    pr = datagen.cfg4()
    rv = RotVote(max_n=pr.n, chain=(15, 45, 180, 360))
    sync = rv.twin(planner="device_sync")
    try:
        a, ma = solve_all(torch_cuda, rv, pr)
        b, mb = solve_all(torch_cuda, sync, pr)
        same(a, b, ma, mb)
        assert a.host_syncs == 1 and not a.flags & RV_RETRIED
        assert a.votes == 10605
    finally:
        rv.close()
        sync.close()


def test_graph_replay_equals_direct(torch_cuda):
    """The second solve with the same (x, y, n, eps, levels, mask) is captured as a CUDA graph
    and later ones replay it: every solve must return the first (directly enqueued) result bit
    for bit; a new mask buffer or eps starts over (direct, capture, replay)."""
    from paper_2506_11547_b200 import RotVote
    pr = datagen.make_problem(20000, 400, 0.01, 0.05, seed=21)
    rv = RotVote(max_n=pr.n)
    try:
        x, y = dev(torch_cuda, pr.x), dev(torch_cuda, pr.y)
        mask = torch_cuda.zeros((pr.n + 31) // 32, dtype=torch_cuda.int32, device="cuda")
        ref = rv.solve(x, y, pr.eps, mask=mask)
        m_ref = mask.cpu().numpy()
        for k in range(4):
            mask.zero_()
            r = rv.solve(x, y, pr.eps, mask=mask)
            same(r, ref, mask.cpu().numpy(), m_ref)
            assert r.host_syncs == 1 and r.launches == ref.launches, (k, r.host_syncs, r.launches)
            assert abs(sum(r.phase_ms.values()) - r.ms) <= 0.05 * r.ms + 0.05
        mask2 = torch_cuda.zeros_like(mask)
        for k in range(3):
            r = rv.solve(x, y, pr.eps, mask=mask2)
            same(r, ref, mask2.cpu().numpy(), m_ref)
        r = rv.solve(x, y, pr.eps * 1.2, mask=mask2)  # another key: direct again
        ref2 = rv.twin(planner="device_sync").solve(x, y, pr.eps * 1.2)
        assert (r.cell, r.votes, r.n_tied) == (ref2.cell, ref2.votes, ref2.n_tied)
        assert np.array_equal(r.q, ref2.q)
    finally:
        rv.close()


@pytest.mark.parametrize("chain", [(15, 45, 180, 360), (15, 45, 90, 180, 360),
                                   (5, 15, 45, 90, 180, 360), (15, 45, 360)])
def test_one_pass_chains_no_retry(torch_cuda, chain):
    """Resolution chains with every dive-level size (f = 2, 3, 4, 8): the one-pass solve must
    finish in one pass (a retry would hide a broken one-pass level behind the per-level loop's
    correct answer) and equal the per-level loop bit for bit."""
    from paper_2506_11547_b200 import RotVote
    pr = datagen.make_problem(30000, 600, 0.01, 0.05, seed=17)
    rv = RotVote(max_n=pr.n, chain=chain)
    sync = rv.twin(planner="device_sync")
    try:
        a, ma = solve_all(torch_cuda, rv, pr)
        b, mb = solve_all(torch_cuda, sync, pr)
        same(a, b, ma, mb)
        assert a.host_syncs == 1 and not a.flags & RV_RETRIED, (a.host_syncs, a.flags)
    finally:
        rv.close()
        sync.close()
