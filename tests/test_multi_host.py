"""NEXT-2 (several rotations) on CPU: the host planner with exclusion balls,
driven by exact oracle counts, finds the oracle's greedy peaks (the plain definition,
oracle.solve_multi: exact counts of every finest block, then suppression of the blocks
within rho of each earlier peak) -- cell, votes and ties, for random chains, `levels`,
suppression angles and two-structure scenes."""
import numpy as np
import pytest

import datagen
import oracle
from paper_2506_11547_b200 import rotvote as rvmod
from planner_util import run_plan


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2506_11547_b200 import build
    build.build()
    oracle.build()


CHAINS = [(5, 15, 45), (3, 9, 27), (4, 8, 16, 32), (6, 18)]


def _multi_by_planner(x, y, eps, chain, levels, K, rho):
    peaks = []
    for _ in range(K):
        excl = np.array([oracle.cell_quat(chain[-1], p[0]) for p in peaks]).reshape(-1, 4)
        r = run_plan(x, y, eps, chain, levels, excl=excl, rho=rho)
        if r.votes == 0 and r.n_tied == 0:
            break
        peaks.append((r.lin, r.votes, r.n_tied))
    return peaks


def test_planner_with_exclusions_equals_greedy_definition():
    rng = np.random.default_rng(12)
    for trial in range(16):
        n = int(rng.integers(20, 160))
        eps = float(rng.choice([0.05, 0.1, 0.3]))
        pr = datagen.make_problem(n, n // 3, 0.01, eps, seed=int(rng.integers(1 << 30)),
                                  n_inl2=n // 4, sigma2=0.01)
        chain = CHAINS[trial % len(CHAINS)]
        rho = float(rng.choice([0.05, 0.2, 0.6]))
        K = 3
        ref = oracle.solve_multi(pr.x, pr.y, eps, chain[-1], K, rho)
        for L in sorted({1, 2, len(chain)}):
            got = _multi_by_planner(pr.x, pr.y, eps, chain, L, K, rho)
            assert got == [(o[0], o[1], o[2]) for o in ref], (trial, chain, L, rho)


def test_two_structures_are_both_found():
    """the inliers of two rotations give two peaks.  The two peaks are R and R2
    (in either order: which is fuller depends on where the block centres fall), each within
    the grid's resolution (B = 90: block half-diagonal ~4.4 degrees of rotation)."""
    from scipy.spatial.transform import Rotation as Rot
    pr = datagen.make_problem(400, 80, 0.005, 0.08, seed=99, n_inl2=60, sigma2=0.005)
    chain = (5, 15, 45, 90)
    peaks = _multi_by_planner(pr.x, pr.y, 0.08, chain, 4, 2, 0.3)
    assert len(peaks) == 2
    ang = np.zeros((2, 2))
    for a_, (lin, votes, _) in enumerate(peaks):
        w, a, b, c = oracle.cell_quat(90, lin)
        for b_, R in enumerate((pr.R, pr.R2)):
            ang[a_, b_] = np.degrees((Rot.from_matrix(R).inv() *
                                      Rot.from_quat([a, b, c, w])).magnitude())
    assert min(ang[0, 0] + ang[1, 1], ang[0, 1] + ang[1, 0]) < 2 * 4.5
    assert ang.min(axis=0).max() < 4.5


def test_everything_excluded_gives_no_peak():
    pr = datagen.make_problem(50, 10, 0.01, 0.1, seed=4)
    q = oracle.cell_quat(15, 0)
    r = run_plan(pr.x, pr.y, 0.1, (5, 15), 2, excl=np.array([q]), rho=np.pi)
    assert (r.votes, r.n_tied) == (0, 0)


def test_bad_exclusion_arguments():
    with pytest.raises(ValueError):
        rvmod.Plan((5, 15), 2, 10, 0.1, excl=np.zeros((1, 4)), rho=0.2)   # zero quaternion
    with pytest.raises(ValueError):
        rvmod.Plan((5, 15), 2, 10, 0.1, excl=np.array([[1.0, 0, 0, 0]]), rho=4.0)
