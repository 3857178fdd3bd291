"""NEXT-2: several rotations (rot_vote_solve_multi) against the oracle's plain definition
(oracle.solve_multi: exact counts of every finest block, greedy peaks with suppression) --
cell, votes and ties of every peak, refined rotations against the oracle's refinement, K = 1
against rot_vote_solve, and the two structures of BASELINE config 3."""
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


@pytest.mark.parametrize("tensor_vote", [False, True])
@pytest.mark.parametrize("chain", [(5, 15, 45), (5, 15, 45, 90)])
def test_multi_equals_greedy_definition(torch_cuda, chain, tensor_vote):
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    rng = np.random.default_rng(len(chain) + 10 * tensor_vote)
    ctx = RotVote(max_n=4096, chain=chain, tensor_vote=tensor_vote)
    try:
        for trial in range(4):
            n = int(rng.integers(100, 1500))
            eps = float(rng.choice([0.05, 0.1]))
            pr = datagen.make_problem(n, n // 5, 0.01, eps, seed=int(rng.integers(1 << 30)),
                                      n_inl2=n // 8, sigma2=0.01)
            rho = float(rng.choice([0.1, 0.4]))
            got = ctx.solve_multi(dev(torch, pr.x), dev(torch, pr.y), eps, 3, rho,
                                  levels=len(chain))
            ref = oracle.solve_multi(pr.x, pr.y, eps, chain[-1], 3, rho)
            assert [(g.lin, g.votes, g.n_tied) for g in got] == [o[:3] for o in ref]
            for g in got:
                q, fl, _ = oracle.refine(pr.x, pr.y, eps, g.q_cell)
                assert oracle.rotation_angle_between(g.q, q) < 1e-9
    finally:
        ctx.close()


def test_multi_k1_equals_solve(torch_cuda):
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    ctx = RotVote(max_n=1 << 17)
    try:
        for pr in (datagen.cfg1(), datagen.cfg2(seed=2)):
            x, y = dev(torch, pr.x), dev(torch, pr.y)
            m = ctx.solve_multi(x, y, pr.eps, 1, 0.2)
            s = ctx.solve(x, y, pr.eps)
            assert len(m) == 1
            assert (m[0].cell, m[0].votes, m[0].n_tied) == (s.cell, s.votes, s.n_tied)
            assert np.array_equal(m[0].q, s.q)
    finally:
        ctx.close()


def test_multi_config3_finds_both_structures(torch_cuda):
    """BASELINE config 3: 5% inliers to R, 3% to an independent R2 (the paper's multiple
    rotations): the first two peaks, refined, are R and R2."""
    from paper_2506_11547_b200 import RotVote
    torch = torch_cuda
    pr = datagen.cfg3()
    ctx = RotVote(max_n=pr.n)
    try:
        got = ctx.solve_multi(dev(torch, pr.x), dev(torch, pr.y), pr.eps, 2, 0.2)
        assert len(got) == 2
        errs = [np.degrees(oracle.rotation_angle_between(g.q, _quat(R)))
                for g, R in zip(got, (pr.R, pr.R2))]
        assert max(errs) < 0.5, errs
        assert got[0].votes > got[1].votes
    finally:
        ctx.close()


def _quat(R):
    from scipy.spatial.transform import Rotation
    x, y, z, w = Rotation.from_matrix(R).as_quat()
    return np.array([w, x, y, z])


def test_multi_rejects_bad_arguments(torch_cuda):
    from paper_2506_11547_b200 import RotVote, RotVoteError
    torch = torch_cuda
    pr = datagen.cfg1()
    ctx = RotVote(max_n=1024)
    try:
        x, y = dev(torch, pr.x), dev(torch, pr.y)
        for K, rho in ((0, 0.2), (65, 0.2), (2, -0.1), (2, 3.5)):
            with pytest.raises(RotVoteError):
                ctx.solve_multi(x, y, pr.eps, K, rho)
        assert len(ctx.solve_multi(x, y, pr.eps, 2, 0.2)) == 2
    finally:
        ctx.close()
