"""CPU pins of the ancestor-culling certificate ("Ancestor culling").

The culled vote counts a block c only over the correspondences that pass the bound test of its
level-0 ancestor a.  That is exact iff every correspondence that can vote for c (exact
s_i(q_c) >= cos(eps + r(c)) at a bound level, s_i(q_c) >= cos(eps) at the final level) also has
s_i(q_a) >= cos(eps + r(a)).  The argument is R6's triangle inequality on nested boxes:
  (1) geometric: r(a) >= r(c) + 2 lambda(a) |p_c - p_a| for every block c inside a, with
      r = 2 lambda sqrt(3)/B the oracle's bound radius;
  (2) the rotation distance between q_c and q_a is at most 2 lambda(a) |p_c - p_a|;
  (3) hence the implication above, checked here by brute force on random data with the
      oracle's exact statistic (no GPU code involved).
"""
import math

import numpy as np
import pytest

import datagen
import oracle


@pytest.fixture(scope="module", autouse=True)
def built():
    oracle.build()


def _ijk(B, lin):
    lin = int(lin)
    return lin // (B * B), (lin // B) % B, lin % B


def _lam_max(B, i, j, k):
    """largest conformal factor 2 / (1 + |p|^2) of P' over the block (at its point nearest the
    origin), in double"""
    lo = np.array([(2 * v - B) / B for v in (i, j, k)])
    hi = lo + 2.0 / B
    d = np.where(lo > 0, lo, np.where(hi < 0, -hi, 0.0))
    return 2.0 / (1.0 + float(d @ d))


@pytest.mark.parametrize("B0,f", [(15, 3), (15, 6), (15, 24), (5, 3), (5, 9), (45, 2)])
def test_ancestor_radius_covers_child(B0, f):
    """(1): r(a) >= r(c) + 2 lambda(a) |p_c - p_a| for children / descendants of random
    ancestors (nested grids B = f B0)."""
    B = f * B0
    rng = np.random.default_rng(B0 * 100 + f)
    anc = oracle.candidates(B0)
    for a in rng.choice(anc, min(60, anc.size), replace=False):
        ai, aj, ak = _ijk(B0, a)
        ra = oracle.cell_radius(B0, ai, aj, ak)
        pa = oracle.cell_center(B0, ai, aj, ak)
        lam = _lam_max(B0, ai, aj, ak)
        for _ in range(20):
            ci, cj, ck = (f * ai + rng.integers(f), f * aj + rng.integers(f), f * ak + rng.integers(f))
            if not oracle.cell_is_candidate(B, ci, cj, ck):
                continue
            rc = oracle.cell_radius(B, ci, cj, ck)
            pc = oracle.cell_center(B, ci, cj, ck)
            assert rc + 2.0 * lam * np.linalg.norm(pc - pa) <= ra * (1 + 1e-12), (a, ci, cj, ck)


def test_rotation_distance_within_conformal_bound():
    """(2): the rotation angle between q_c and q_a is <= 2 lambda(a) |p_c - p_a|."""
    rng = np.random.default_rng(1)
    B0, f = 15, 3
    for a in rng.choice(oracle.candidates(B0), 200, replace=False):
        ai, aj, ak = _ijk(B0, a)
        qa = oracle.cell_quat(B0, int(a))
        lam = _lam_max(B0, ai, aj, ak)
        pa = oracle.cell_center(B0, ai, aj, ak)
        for _ in range(10):
            ci, cj, ck = f * ai + rng.integers(f), f * aj + rng.integers(f), f * ak + rng.integers(f)
            if not oracle.cell_is_candidate(B0 * f, ci, cj, ck):
                continue
            lin = oracle.lin_of(B0 * f, ci, cj, ck)
            qc = oracle.cell_quat(B0 * f, lin)
            pc = oracle.cell_center(B0 * f, ci, cj, ck)
            ang = oracle.rotation_angle_between(qa, qc)
            assert ang <= 2.0 * lam * np.linalg.norm(pc - pa) + 1e-12


@pytest.mark.parametrize("eps", [0.05, 0.2, 1.0])
def test_every_voter_of_a_child_passes_its_ancestor(eps):
    """(3) by brute force: over random correspondences (inliers of a random rotation plus
    outliers) and random blocks at B = 45 and 360, every i with s_i(q_c) >= cos(eps + r(c))
    (bound level) or >= cos(eps) (final level) has s_i(q_a) >= cos(eps + r(a)), B0 = 15."""
    pr = datagen.make_problem(4000, 1000, 0.01, eps, seed=3)
    rng = np.random.default_rng(7)
    B0 = 15
    # blocks near the truth (many voters) and random ones
    for B in (45, 360):
        cand = oracle.candidates(B)
        lins = list(rng.choice(cand, 40, replace=False))
        ref = oracle.solve(pr.x, pr.y, eps) if B == 360 else None
        if ref is not None:
            lins.append(ref.lin)
        for lin in lins:
            ci, cj, ck = _ijk(B, lin)
            f = B // B0
            a = oracle.lin_of(B0, ci // f, cj // f, ck // f)
            sa = oracle.pair_stats(pr.x, pr.y, oracle.cell_quat(B0, a))
            sc = oracle.pair_stats(pr.x, pr.y, oracle.cell_quat(B, lin))
            ta = oracle.cell_bound_threshold(B0, a, eps)
            tc = oracle.cell_bound_threshold(B, lin, eps)
            for t in (tc, math.cos(eps)):
                voters = sc >= t
                assert np.all(sa[voters] >= ta), (B, lin)
