"""Ancestor culling (K3-TC bitmasks + K3-C, csrc/rv_cull.cu) against the oracle.

The culled vote counts a block only over the correspondences that passed its level-0
ancestor's bound test.  The bar is the one of every count in this repo: each
(block, correspondence) pair more than 1e-5 from the threshold in use is decided as the
oracle decides it, so
  * the level-0 bitmask bit of (a, i) is 1 when s_i(q_a) >= t'(a) + 1e-5 and 0 when
    s_i(q_a) < t'(a) - 1e-5 (t' = the K3-TC bound threshold, guard 1e-5 + 1.5e-5);
  * a culled count lies in [#{s >= t + 1e-5}, #{s >= t - 1e-5}] for the threshold t of its
    mode -- and, since culled pairs are evaluated with K3's exact arithmetic, it never exceeds
    the unculled FP32 count of the same block;
  * whole solves return the oracle's (cell, votes, ties) and a rotation within 1e-4 rad, and
    exactly the unculled solve's result.
"""
import math

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu
BAND = 1e-5
GUARD = 1e-5
GUARD_TC = 1e-5 + 1.5e-5
RV_MODE_BOUND, RV_MODE_FINAL = 0, 1


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _ctx(path, **kw):
    """A culling context on the tensor-core K3-CT path ("tc", default) or the FP32 K3-C path
    ("fp32", cull = 2)."""
    from paper_2506_11547_b200 import RotVote
    return RotVote(tensor_vote=True, cull=path, **kw)


@pytest.fixture(scope="module", params=["tc", "fp32"])
def rvc(request, torch_cuda):
    from paper_2506_11547_b200 import build
    build.build()
    oracle.build()
    ctx = _ctx(request.param, max_n=1 << 20, max_problems=512)
    ctx.path = request.param
    yield ctx
    ctx.close()


def guard_of(ctx):
    """the guard of a culled count's threshold: K3-CT = K3-TC's, K3-C = K3's"""
    return GUARD_TC if ctx.path == "tc" else GUARD


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def in_band(got, x, y, B, lins, thr):
    """got within [#{s >= thr + band}, #{s >= thr - band}] (oracle, fp64)."""
    ge, near = oracle.count_cells(x, y, B, lins, thr, BAND)
    ge = ge.astype(np.int64)
    near = near.astype(np.int64)
    got = np.asarray(got, np.int64)
    return (got >= ge - near) & (got <= ge + near)


@pytest.mark.parametrize("n,eps,B0", [(3000, 0.05, 15), (1001, 0.3, 15), (20001, 0.08, 15),
                                      (257, 1.2, 5)])
def test_level0_bitmasks_match_oracle(rvc, torch_cuda, n, eps, B0):
    torch = torch_cuda
    pr = datagen.make_problem(n, n // 8, 0.01, eps, seed=n)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    _, bits = rvc.count_cells_culled(x, y, B0, 3 * B0, [], eps, RV_MODE_BOUND, want_bits=True)
    cands = oracle.candidates(B0)
    assert bits.shape == (len(cands), (n + 255) // 256 * 8)
    rng = np.random.default_rng(n)
    rows = rng.choice(len(cands), min(64, len(cands)), replace=False)
    for a in rows:
        lin = int(cands[a])
        s = oracle.pair_stats(pr.x, pr.y, oracle.cell_quat(B0, lin))
        t = oracle.cell_bound_threshold(B0, lin, eps) - GUARD_TC
        w = bits[a]
        b = (w[np.arange(n) // 32] >> (np.arange(n) % 32).astype(np.uint32)) & 1
        assert np.all(b[s >= t + BAND] == 1), a
        assert np.all(b[s < t - BAND] == 0), a
        # columns past n (padding rows) never pass
        tail = np.arange(n, w.size * 32)
        assert np.all(((w[tail // 32] >> (tail % 32).astype(np.uint32)) & 1) == 0)


@pytest.mark.parametrize("n,eps", [(3000, 0.05), (1001, 0.3), (20001, 0.08), (70000, 0.05), (30000, 1.0)])
def test_culled_counts_in_band(rvc, torch_cuda, n, eps):
    """Blocks at B = 45, 90, 360 (random order, repeated blocks, ragged n) over B0 = 15."""
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    pr = datagen.make_problem(n, n // 10, 0.01, eps, seed=n + 1)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    rng = np.random.default_rng(n)
    fp32 = RotVote(max_n=1 << 20, tensor_vote=False)
    try:
        for B in (45, 90, 360):
            c = oracle.candidates(B)
            lins = rng.choice(c, 300, replace=True).astype(np.uint32)
            lins = np.concatenate([lins, lins[:7]])  # repeats
            g = guard_of(rvc)
            got = rvc.count_cells_culled(x, y, 15, B, lins, eps, RV_MODE_BOUND)
            thr = np.array([oracle.cell_bound_threshold(B, int(l), eps) - g for l in lins])
            assert np.all(in_band(got, pr.x, pr.y, B, lins, thr)), B
            if rvc.path == "fp32":  # a subset evaluated with K3's exact arithmetic
                ref = fp32.count_cells(x, y, B, lins, eps, RV_MODE_BOUND)
                assert np.all(got <= ref), B
            ga, gb = rvc.count_cells_culled(x, y, 15, B, lins, eps, RV_MODE_FINAL)
            tau = math.cos(eps)
            assert np.all(in_band(ga, pr.x, pr.y, B, lins, tau - g)), B
            assert np.all(in_band(gb, pr.x, pr.y, B, lins, tau + g)), B
            if rvc.path == "fp32":
                ra, rb = fp32.count_cells(x, y, B, lins, eps, RV_MODE_FINAL)
                assert np.all(ga <= ra) and np.all(gb <= rb), B
            ex, _ = oracle.count_cells(pr.x, pr.y, B, lins, tau, 0.0)
            assert np.all(gb <= ex) and np.all(ex <= ga), B  # cnt_b <= exact <= cnt_a
    finally:
        fp32.close()


def test_culled_counts_near_the_peak(rvc, torch_cuda):
    """The blocks around the true rotation (long runs of one ancestor, full items)."""
    torch = torch_cuda
    pr = datagen.make_problem(50_000, 2_000, 0.01, 0.05, seed=3)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    ref = oracle.solve(pr.x, pr.y, pr.eps)
    i, j, k = ref.cell
    for B in (45, 90, 360):
        ci, cj, ck = (int(i * B // 360), int(j * B // 360), int(k * B // 360))
        lins = []
        for a in range(-2, 3):
            for b in range(-2, 3):
                for c in range(-2, 3):
                    u, v, w = ci + a, cj + b, ck + c
                    if 0 <= min(u, v, w) and max(u, v, w) < B and oracle.cell_is_candidate(B, u, v, w):
                        lins.append(oracle.lin_of(B, u, v, w))
        lins = np.array(sorted(lins), np.uint32)
        got = rvc.count_cells_culled(x, y, 15, B, lins, pr.eps, RV_MODE_BOUND)
        thr = np.array([oracle.cell_bound_threshold(B, int(l), pr.eps) - guard_of(rvc)
                        for l in lins])
        assert np.all(in_band(got, pr.x, pr.y, B, lins, thr)), B
        assert got.max() >= 2_000 * 0.9, (B, got.max())


def _problems():
    out = [datagen.cfg1(), datagen.cfg2(seed=2), datagen.make_problem(2, 2, 0.0, 0.1, seed=1),
           datagen.make_problem(3, 0, 0.0, 0.5, seed=2),
           datagen.make_problem(5000, 50, 0.02, 0.08, seed=4, n_inl2=30, sigma2=0.02)]
    # y = x and y = -x rows (a = +-b) mixed in
    pr = datagen.make_problem(800, 200, 0.01, 0.05, seed=9)
    pr.y[:5] = pr.x[:5]
    pr.y[5:10] = -pr.x[5:10]
    out.append(pr)
    rng = np.random.default_rng(11)
    for s in range(8):
        n = int(rng.integers(2, 4000))
        out.append(datagen.make_problem(n, int(rng.integers(0, n + 1)), float(rng.uniform(0, 0.03)),
                                        float(rng.choice([0.02, 0.05, 0.1, 0.3, 1.0])), seed=[11, s]))
    return out


def test_culled_solves_match_oracle(rvc, torch_cuda):
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    plain = RotVote(max_n=1 << 20, tensor_vote=True, cull=False)
    try:
        for p, pr in enumerate(_problems()):
            x, y = dev(torch, pr.x), dev(torch, pr.y)
            ref = oracle.solve(pr.x, pr.y, pr.eps)
            for levels in (2, 3, 5, 6, 0):
                r = rvc.solve(x, y, pr.eps, levels=levels)
                assert (r.cell, r.votes, r.n_tied) == (ref.cell, ref.votes, ref.n_tied), (p, levels)
                assert oracle.rotation_angle_between(r.q, ref.q) < 1e-4, (p, levels)
                u = plain.solve(x, y, pr.eps, levels=levels)
                assert (u.cell, u.votes, u.n_tied, u.n_inliers) == (r.cell, r.votes, r.n_tied,
                                                                    r.n_inliers), (p, levels)
                assert np.array_equal(u.q, r.q), (p, levels)
                assert r.pair_votes == sum(c * pr.n for c in r.cells_per_phase), p
            if pr.n >= 1000 and pr.eps <= 0.1:  # levels = 0 (B0 = 15): lists sparse enough
                assert r.cull_launches > 0 and 0 < r.cull_pairs < r.pair_votes, p
    finally:
        plain.close()


def test_culled_batched_matches_oracle(rvc, torch_cuda):
    """A ragged batch (n = 2 ... 2500) through the device level loop with culling."""
    torch = torch_cuda
    rng = np.random.default_rng(5)
    probs = []
    for p in range(96):
        n = int(rng.integers(2, 2500))
        probs.append(datagen.make_problem(n, int(rng.integers(0, n + 1)), float(rng.uniform(0, 0.03)),
                                          0.09, seed=[5, p]))
    bt = datagen.batch_of(probs, 0.09)
    x, y = dev(torch, bt.x), dev(torch, bt.y)
    res = rvc.solve_batched(x, y, bt.offsets, bt.eps)
    for p, pr in enumerate(probs):
        ref = oracle.solve(pr.x, pr.y, bt.eps)
        r = res[p]
        assert (r.cell, r.votes, r.n_tied) == (ref.cell, ref.votes, ref.n_tied), p
        assert oracle.rotation_angle_between(r.q, ref.q) < 1e-4, p


def test_culled_loopback_shards(torch_cuda):
    """emulate_world: level 0 sliced over the emulated ranks with its bitmasks (K3-CT: slices
    at i-slab boundaries, so a rank holds every member of the ancestor groups it owns; K3-C:
    uniform slices), finer levels voted by the owning rank -- the same result and per-phase
    block counts as one rank, on both culled vote paths; the two paths reach the same answer."""
    torch = torch_cuda
    for pr in (datagen.cfg2(seed=5), datagen.make_problem(40_000, 400, 0.01, 0.05, seed=8)):
        x, y = dev(torch, pr.x), dev(torch, pr.y)
        o = oracle.solve(pr.x, pr.y, pr.eps)
        refs = {}
        for path in ("tc", "fp32"):
            ref = None
            for W in (1, 2, 3, 8):
                ctx = _ctx(path, max_n=1 << 17, emulate_world=W)
                try:
                    r = ctx.solve(x, y, pr.eps)
                finally:
                    ctx.close()
                if path == "tc":
                    assert r.cull_tc_launches > 0, W
                if ref is None:
                    ref = r
                    assert (r.cell, r.votes, r.n_tied) == (o.cell, o.votes, o.n_tied)
                assert (r.cell, r.votes, r.n_tied, r.n_inliers) == (ref.cell, ref.votes,
                                                                    ref.n_tied, ref.n_inliers), W
                assert np.array_equal(r.q, ref.q), W
                assert r.cells_per_phase == ref.cells_per_phase, (path, W)
            refs[path] = ref
        a, b = refs["tc"], refs["fp32"]
        assert (a.cell, a.votes, a.n_tied, a.n_inliers) == (b.cell, b.votes, b.n_tied, b.n_inliers)
        assert oracle.rotation_angle_between(a.q, b.q) < 1e-9


def test_culled_chains_agree(torch_cuda):
    """The certified result does not depend on the resolution chain: the bench's chain
    15-45-180-360 and the library's default 15-45-90-180-360 give the oracle's answer on the
    culled tensor-core path."""
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    pr = datagen.make_problem(60_000, 600, 0.01, 0.05, seed=11)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    o = oracle.solve(pr.x, pr.y, pr.eps)
    res = []
    for chain in ((15, 45, 180, 360), None):
        ctx = RotVote(max_n=1 << 17, chain=chain) if chain else RotVote(max_n=1 << 17)
        try:
            r = ctx.solve(x, y, pr.eps, levels=len(chain) if chain else 0)
        finally:
            ctx.close()
        assert r.cull_tc_launches > 0
        assert (r.cell, r.votes, r.n_tied) == (o.cell, o.votes, o.n_tied), chain
        res.append(r)
    assert np.array_equal(res[0].q, res[1].q)
