"""GPU parity: every step of the CUDA path (through the C-ABI) against the CPU oracle.

These tests pin the FP32-pipe vote kernel (K3, contexts with tensor_vote=False); the
tensor-core path (K3-TC, the default) has its own file, test_gpu_tc.py, and the solves there
and in test_gpu_fullsize.py run the default path.

Bar (BASELINE north_star):
  * counts: every (cell, correspondence) pair more than 1e-5 from the threshold in use is
    decided identically -> GPU count in [#{s >= t + 1e-5}, #{s >= t - 1e-5}] (oracle, fp64);
  * exact counts (fp64 recheck) and the winning (cell, votes) identical to the oracle;
  * rotation within 1e-4 rad geodesic of the oracle's (4 asin(|dq|/2));
  * K entries within fp32 rounding of the oracle's Appendix-A matrix.
"""
import math

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

BAND = 1e-5
GUARD = 1e-5


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
    ctx = RotVote(device=0, max_n=4096 * 1000 + 4096, max_problems=4096, tensor_vote=False)
    yield ctx
    ctx.close()


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def in_band_bounds(x, y, B, lins, thr):
    lo, _ = oracle.count_cells(x, y, B, lins, np.asarray(thr) + BAND, band=0)
    hi, _ = oracle.count_cells(x, y, B, lins, np.asarray(thr) - BAND, band=0)
    return lo, hi


def test_setup_matches_appendix_A(rv, torch_cuda):
    torch = torch_cuda
    for n in (1, 2, 257, 1001):
        pr = datagen.make_problem(max(n, 2), max(n, 2) // 2, 0.02, 0.1, seed=n)
        x, y = pr.x[:n] * np.float32(3.5), pr.y[:n] * np.float32(0.25)   # any nonzero length
        k = rv.setup(dev(torch, x), dev(torch, y)).cpu().numpy().astype(np.float64)
        xn = x.astype(np.float64); xn /= np.linalg.norm(xn, axis=1, keepdims=True)
        yn = y.astype(np.float64); yn /= np.linalg.norm(yn, axis=1, keepdims=True)
        for i in range(n):
            M = oracle.constraint_M(xn[i], yn[i])
            want = [M[0, 0], M[1, 1], M[2, 2], M[0, 1], M[0, 2], M[0, 3], M[1, 2], M[1, 3], M[2, 3]]
            assert np.allclose(k[:, i], want, rtol=0, atol=1.2e-7), i
            assert abs(M[3, 3] + M[0, 0] + M[1, 1] + M[2, 2]) < 1e-14


def _sample_cells(rng, B, m):
    cand = oracle.candidates(B)
    return np.sort(rng.choice(cand, size=min(m, cand.size), replace=False)).astype(np.uint32)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_count_cells_bound_mode(rv, torch_cuda, cfg):
    from paper_2506_11547_b200 import RV_MODE_BOUND
    torch = torch_cuda
    pr = datagen.CONFIGS[cfg]()
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    rng = np.random.default_rng(1)
    for B in (5, 15, 45, 90):
        lins = _sample_cells(rng, B, 700)
        got = rv.count_cells(x, y, B, lins, pr.eps, RV_MODE_BOUND)
        thr = np.array([oracle.cell_bound_threshold(B, int(l), pr.eps) for l in lins]) - GUARD
        lo, hi = in_band_bounds(pr.x, pr.y, B, lins, thr)
        assert np.all(got >= lo) and np.all(got <= hi), B
        # non-vacuity: most cells have an empty near band.  Outlier scores are uniform on
        # [-1, 1] (Archimedes), so P(|s - t| < g) = g per pair and a cell's band
        # is empty with probability ~exp(-n g): 0.999 at cfg1, 0.905 at cfg2 (5 sigma of
        # 700 cells below that is 0.056)
        assert np.mean(lo == hi) >= math.exp(-pr.n * GUARD) - 0.06


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_count_cells_final_and_exact(rv, torch_cuda, cfg):
    from paper_2506_11547_b200 import RV_MODE_EXACT, RV_MODE_FINAL
    torch = torch_cuda
    pr = datagen.CONFIGS[cfg]()
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    rng = np.random.default_rng(2)
    tau = math.cos(pr.eps)
    # random cells plus the neighbourhood of the oracle's winner (where counts are large)
    ref = oracle.solve(pr.x, pr.y, pr.eps)
    i, j, k = ref.cell
    near = [oracle.lin_of(360, i + a, j + b, k + c) for a in (-2, 0, 2) for b in (-2, 0, 2)
            for c in (-2, 0, 2)]
    lins = np.unique(np.concatenate([_sample_cells(rng, 360, 500), near]).astype(np.uint32))
    a, b = rv.count_cells(x, y, 360, lins, pr.eps, RV_MODE_FINAL)
    lo, hi = in_band_bounds(pr.x, pr.y, 360, lins, tau - GUARD)
    assert np.all(a >= lo) and np.all(a <= hi)
    lo, hi = in_band_bounds(pr.x, pr.y, 360, lins, tau + GUARD)
    assert np.all(b >= lo) and np.all(b <= hi)
    assert np.all(b <= a)
    ex = rv.count_cells(x, y, 360, lins, pr.eps, RV_MODE_EXACT)
    want, near_cnt = oracle.count_cells(pr.x, pr.y, 360, lins, tau, band=1e-12)
    ok = near_cnt == 0
    assert np.array_equal(ex[ok], want[ok])
    assert np.all(ex >= b) and np.all(ex <= a)


def test_count_cells_ragged_and_many_tiles(rv, torch_cuda):
    """N not a multiple of the tile / of 4; cells spanning several CTAs; eps large enough
    that thresholds go negative (zero-padding rows must not be counted)."""
    from paper_2506_11547_b200 import RV_MODE_BOUND, RV_MODE_EXACT, RV_MODE_FINAL
    torch = torch_cuda
    rng = np.random.default_rng(3)
    for n, eps in ((3, 0.3), (257, 2.0), (1001, 1.7), (4099, 0.05), (70001, 0.2)):
        pr = datagen.make_problem(n, n // 3, 0.02, eps, seed=n)
        x, y = dev(torch, pr.x), dev(torch, pr.y)
        for B, mode in ((5, RV_MODE_BOUND), (15, RV_MODE_BOUND), (45, RV_MODE_FINAL),
                        (90, RV_MODE_EXACT)):
            lins = _sample_cells(rng, B, 2500)
            got = rv.count_cells(x, y, B, lins, eps, mode)
            tau = math.cos(eps)
            if mode == RV_MODE_BOUND:
                thr = np.array([oracle.cell_bound_threshold(B, int(l), eps) for l in lins]) - GUARD
                lo, hi = in_band_bounds(pr.x, pr.y, B, lins, thr)
                assert np.all(got >= lo) and np.all(got <= hi), (n, B)
            elif mode == RV_MODE_FINAL:
                a, b = got
                lo, hi = in_band_bounds(pr.x, pr.y, B, lins, tau - GUARD)
                assert np.all(a >= lo) and np.all(a <= hi), (n, B)
                lo, hi = in_band_bounds(pr.x, pr.y, B, lins, tau + GUARD)
                assert np.all(b >= lo) and np.all(b <= hi), (n, B)
            else:
                want, nr = oracle.count_cells(pr.x, pr.y, B, lins, tau, band=1e-12)
                assert np.array_equal(got[nr == 0], want[nr == 0]), (n, B)


def check_solution(res, ref, B=360):
    assert res.B == B == ref.B
    assert (res.cell, res.votes, res.n_tied) == (ref.cell, ref.votes, ref.n_tied)
    assert oracle.rotation_angle_between(res.q_cell, ref.q_cell) < 1e-12
    assert oracle.rotation_angle_between(res.q, ref.q) < 1e-4
    assert res.flags & 3 == ref.flags & 3


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_solve_matches_oracle(rv, torch_cuda, cfg):
    from paper_2506_11547_b200 import unpack_mask
    torch = torch_cuda
    pr = datagen.CONFIGS[cfg]()
    ref = oracle.solve(pr.x, pr.y, pr.eps)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    mask = torch.zeros((pr.n + 31) // 32, dtype=torch.int32, device="cuda")
    res = rv.solve(x, y, pr.eps, mask=mask)
    check_solution(res, ref)
    assert oracle.rotation_angle_between(res.q, ref.q) < 1e-9
    m = unpack_mask(mask.cpu().numpy(), pr.n)
    s = oracle.pair_stats(pr.x, pr.y, res.q)
    far = np.abs(s - math.cos(pr.eps)) > 1e-9
    assert np.array_equal(m[far], ref.mask[far])
    assert res.n_inliers == int(m.sum())
    # the paper's success criterion (e_R <= 5 deg) against the ground truth
    from scipy.spatial.transform import Rotation as Rot
    eR = np.degrees(Rot.from_matrix(pr.R.T @ oracle.quat_to_R(res.q)).magnitude())
    assert eR < 1.0


def test_levels_do_not_change_the_result(rv, torch_cuda):
    torch = torch_cuda
    pr = datagen.cfg2()
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    base = rv.solve(x, y, pr.eps)
    for L in (1, 2, 3, 4, 5, 6):
        r = rv.solve(x, y, pr.eps, levels=L)
        assert (r.cell, r.votes, r.n_tied) == (base.cell, base.votes, base.n_tied), L
        assert np.array_equal(r.q, base.q)
    assert rv.solve(x, y, pr.eps, levels=1).cells_evaluated == 24733672


def test_loopback_sharding_is_invariant(torch_cuda):
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    pr = datagen.cfg2(seed=5)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    outs = []
    for W in (1, 2, 3, 8):
        ctx = RotVote(max_n=1 << 16, emulate_world=W, tensor_vote=False)
        outs.append(ctx.solve(x, y, pr.eps))
        ctx.close()
    for r in outs[1:]:
        assert (r.cell, r.votes, r.n_tied, r.pair_votes) == (outs[0].cell, outs[0].votes,
                                                             outs[0].n_tied, outs[0].pair_votes)
        assert np.array_equal(r.q, outs[0].q)


def test_refine_matches_oracle(rv, torch_cuda):
    from paper_2506_11547_b200 import unpack_mask
    from scipy.spatial.transform import Rotation as Rot
    torch = torch_cuda
    for seed in range(4):
        pr = datagen.make_problem(30000, 3000, 0.02, 0.07, seed=seed)
        q0 = Rot.from_matrix(pr.R).as_quat(scalar_first=True) + 0.003 * np.random.default_rng(seed).standard_normal(4)
        q0 = q0 / np.linalg.norm(q0)
        x, y = dev(torch, pr.x), dev(torch, pr.y)
        mask = torch.zeros((pr.n + 31) // 32, dtype=torch.int32, device="cuda")
        for rounds in (0, 1, 2, 3):
            q, fl, ni = rv.refine(x, y, pr.eps, q0, rounds=rounds, mask=mask)
            qo, flo, mo = oracle.refine(pr.x, pr.y, pr.eps, q0, rounds=rounds)
            assert oracle.rotation_angle_between(q, qo) < 1e-10
            assert fl == flo
            assert np.array_equal(unpack_mask(mask.cpu().numpy(), pr.n), mo)
            assert ni == int(mo.sum())


def test_solve_host_equals_device(rv, torch_cuda):
    torch = torch_cuda
    pr = datagen.cfg2(seed=7)
    a = rv.solve(dev(torch, pr.x), dev(torch, pr.y), pr.eps)
    mask = np.zeros((pr.n + 31) // 32, np.uint32)
    b = rv.solve_host(pr.x, pr.y, pr.eps, mask=mask)
    assert (a.cell, a.votes) == (b.cell, b.votes) and np.array_equal(a.q, b.q)
    assert int(np.unpackbits(mask.view(np.uint8)).sum()) == b.n_inliers


def test_batched_matches_oracle(rv, torch_cuda):
    from paper_2506_11547_b200 import unpack_mask
    torch = torch_cuda
    probs = []
    rng = np.random.default_rng(9)
    for p in range(40):   # ragged sizes, BASELINE config-5 statistics
        n = int(rng.integers(2, 1500))
        sig = float(rng.uniform(0.005, 0.03))
        probs.append(datagen.make_problem(n, max(0, n // 5), sig, 0.09, seed=[9, p]))
    bt = datagen.batch_of(probs, 0.09)
    x, y = dev(torch, bt.x), dev(torch, bt.y)
    words = sum((p.n + 31) // 32 for p in probs)
    masks = torch.zeros(words, dtype=torch.int32, device="cuda")
    res = rv.solve_batched(x, y, bt.offsets, bt.eps, masks=masks)
    mw = masks.cpu().numpy()
    w = 0
    for p, r in zip(probs, res):
        ref = oracle.solve(p.x, p.y, bt.eps)
        check_solution(r, ref)
        m = unpack_mask(mw[w:w + (p.n + 31) // 32], p.n)
        w += (p.n + 31) // 32
        s = oracle.pair_stats(p.x, p.y, r.q)
        far = np.abs(s - math.cos(bt.eps)) > 1e-9
        assert np.array_equal(m[far], ref.mask[far])


def test_batched_cfg5_equals_single_solves(rv, torch_cuda):
    torch = torch_cuda
    bt = datagen.cfg5()
    x, y = dev(torch, bt.x), dev(torch, bt.y)
    res = rv.solve_batched(x, y, bt.offsets, bt.eps)
    assert len(res) == 4096
    rng = np.random.default_rng(11)
    for p in rng.choice(4096, 12, replace=False):
        pr = bt.problems[p]
        single = rv.solve(dev(torch, pr.x), dev(torch, pr.y), bt.eps)
        assert (res[p].cell, res[p].votes, res[p].n_tied) == (single.cell, single.votes, single.n_tied)
        assert np.array_equal(res[p].q, single.q)
        # the device-side level-0 reduction takes the host planner's decisions
        assert res[p].cells_per_phase == single.cells_per_phase
        ref = oracle.solve(pr.x, pr.y, bt.eps)
        check_solution(res[p], ref)
    from scipy.spatial.transform import Rotation as Rot
    errs = [np.degrees(Rot.from_matrix(pr.R.T @ oracle.quat_to_R(r.q)).magnitude())
            for pr, r in zip(bt.problems, res)]
    assert np.mean(np.array(errs) < 5.0) > 0.99    # success criterion


def test_edge_cases(rv, torch_cuda):
    from paper_2506_11547_b200 import RotVoteError
    from paper_2506_11547_b200.rotvote import RV_EDATA, RV_EINVAL
    torch = torch_cuda
    pr = datagen.make_problem(64, 20, 0.01, 0.05, seed=4)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    with pytest.raises(RotVoteError) as e:
        rv.solve(x[:1], y[:1], 0.05)
    assert e.value.code == RV_EINVAL
    for bad_eps in (0.0, -0.1, math.pi, 4.0, float("nan")):
        with pytest.raises(RotVoteError):
            rv.solve(x, y, bad_eps)
    with pytest.raises(RotVoteError):
        rv.solve(x, y, 0.05, levels=7)
    for val in (0.0, float("nan"), float("inf")):
        xb = pr.x.copy(); xb[17] = val
        with pytest.raises(RotVoteError) as e:
            rv.solve(dev(torch, xb), y, 0.05)
        assert e.value.code == RV_EDATA
    # two exact correspondences: closed-form intersection of two great circles
    q_true = np.array([math.sqrt(.5), 0, 0, math.sqrt(.5)])
    R = np.array([[0.0, -1, 0], [1, 0, 0], [0, 0, 1]])
    x2 = np.array([[0.25, -0.5, 0.75], [0.5, 0.125, -0.625]], np.float32)
    y2 = (R @ x2.astype(float).T).T.astype(np.float32)
    r = rv.solve(dev(torch, x2), dev(torch, y2), 0.05)
    assert r.votes == 2 and oracle.rotation_angle_between(r.q, q_true) < 1e-9
    # y = x (identity) and y = -x rows
    xi = pr.x.copy(); yi = pr.x.copy(); yi[::2] = -xi[::2]
    r = rv.solve(dev(torch, xi), dev(torch, yi), 0.05)
    ref = oracle.solve(xi, yi, 0.05)
    check_solution(r, ref)
    # pure outliers
    out = datagen.make_problem(5000, 0, 0.0, 0.05, seed=6)
    r = rv.solve(dev(torch, out.x), dev(torch, out.y), 0.05)
    ref = oracle.solve(out.x, out.y, 0.05)
    check_solution(r, ref)
    # n > max_n
    from paper_2506_11547_b200 import RotVote
    small = RotVote(max_n=100, tensor_vote=False)
    with pytest.raises(RotVoteError) as e:
        small.solve(x, y, 0.05) if x.shape[0] > 100 else small.solve(
            dev(torch, np.tile(pr.x, (2, 1))), dev(torch, np.tile(pr.y, (2, 1))), 0.05)
    assert e.value.code == RV_EINVAL
    small.close()


def test_determinism(rv, torch_cuda):
    torch = torch_cuda
    pr = datagen.cfg3()
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    a = rv.solve(x, y, pr.eps)
    b = rv.solve(x, y, pr.eps)
    assert (a.cell, a.votes, a.pair_votes) == (b.cell, b.votes, b.pair_votes)
    assert np.array_equal(a.q, b.q)


def test_nccl_path_single_rank(torch_cuda):
    """world = 1 with an NCCL id runs the sharded path through a real 1-rank communicator
    (ncclCommInitRank + ncclAllGather of the counts, dlopen'ed libnccl) and must give the
    same answer as the direct path; batched results go through the result all-gather."""
    from paper_2506_11547_b200 import RotVote, rot_vote_get_unique_id
    torch = torch_cuda
    pr = datagen.cfg2(seed=3)
    x, y = dev(torch, pr.x), dev(torch, pr.y)
    plain = RotVote(max_n=1 << 16, tensor_vote=False)
    viaccl = RotVote(max_n=1 << 16, max_problems=8, nccl_id=rot_vote_get_unique_id(),
                     tensor_vote=False)
    a, b = plain.solve(x, y, pr.eps), viaccl.solve(x, y, pr.eps)
    assert (a.cell, a.votes, a.n_tied, a.pair_votes) == (b.cell, b.votes, b.n_tied, b.pair_votes)
    assert np.array_equal(a.q, b.q)
    probs = [datagen.make_problem(500 + 37 * p, 100, 0.01, 0.05, seed=[4, p]) for p in range(5)]
    bt = datagen.batch_of(probs, 0.05)
    rb = viaccl.solve_batched(dev(torch, bt.x), dev(torch, bt.y), bt.offsets, bt.eps)
    for p, r in zip(probs, rb):
        s = plain.solve(dev(torch, p.x), dev(torch, p.y), bt.eps)
        assert (r.cell, r.votes) == (s.cell, s.votes) and np.array_equal(r.q, s.q)
    plain.close()
    viaccl.close()
