"""Pins of the oracle's Algorithm 1 (NEXT-4) against what the paper and the
mathematics fix -- not against a retyped copy of its formulas:

* the circle basis: q_b1, q_b2 orthonormal, every q(alpha) satisfies the
  constraint b^T R(q) a = 1 for random, equal and antipodal pairs; q_b1 equals the
  paper's [cos(theta/2), sin(theta/2) c] with theta = arccos(a.b) (the half-angle reading
  R13); a = b = e_z gives the rotations about z in closed form;
* the samples: a noise-free inlier circle passes within pi/(2J) (half the sample step in
  quaternion angle) of the true rotation;
* the bins: every sample's projected point lies inside its bin box of the grid
  [-1,1]^3 / B (numpy edges), and every correspondence casts exactly J votes;
* the whole Algorithm 1 on config 1 peaks next to the exact consensus winner.
"""
import numpy as np
import pytest

import datagen
import oracle


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def _unit(v):
    v = np.asarray(v, float)
    return v / np.linalg.norm(v)


def _pairs(rng, k):
    out = []
    for _ in range(k):
        a = _unit(rng.normal(size=3))
        out.append((a, _unit(rng.normal(size=3))))
    a = _unit(rng.normal(size=3))
    out += [(a, a.copy()), (a, -a), (np.array([0, 0, 1.0]), np.array([0, 0, -1.0])),
            (np.array([1.0, 0, 0]), np.array([1.0, 0, 0]))]
    b = _unit(a + 1e-9 * rng.normal(size=3))
    out.append((a, b))
    return out


def test_basis_orthonormal_and_on_the_circle():
    rng = np.random.default_rng(1)
    for a, b in _pairs(rng, 40):
        q1, q2 = oracle.alg1_basis(a, b)
        assert abs(q1 @ q1 - 1) < 1e-12 and abs(q2 @ q2 - 1) < 1e-12 and abs(q1 @ q2) < 1e-12
        for al in np.linspace(-np.pi, np.pi, 13):
            q = q1 * np.cos(al / 2) + q2 * np.sin(al / 2)
            assert abs(oracle.vote_stat(q, a, b) - 1.0) < 1e-12


def test_basis_matches_the_papers_trigonometric_form():
    rng = np.random.default_rng(2)
    for _ in range(50):
        a, b = _unit(rng.normal(size=3)), _unit(rng.normal(size=3))
        th = np.arccos(np.clip(a @ b, -1, 1))
        c = np.cross(a, b) / np.linalg.norm(np.cross(a, b))
        q1_paper = np.concatenate([[np.cos(th / 2)], np.sin(th / 2) * c])
        q123 = q1_paper[1:]
        q2_paper = np.concatenate([[-b @ q123], q1_paper[0] * b + np.cross(b, q123)])
        q1, q2 = oracle.alg1_basis(a, b)
        assert np.allclose(q1, q1_paper, atol=1e-12) and np.allclose(q2, q2_paper, atol=1e-12)


def test_basis_closed_form_rotations_about_z():
    q1, q2 = oracle.alg1_basis([0, 0, 1.0], [0, 0, 1.0])
    for al in np.linspace(-np.pi, np.pi, 9):
        q = q1 * np.cos(al / 2) + q2 * np.sin(al / 2)
        assert np.allclose(q, [np.cos(al / 2), 0, 0, np.sin(al / 2)], atol=1e-15)


def _quat(R):
    """scalar-first unit quaternion of R (scipy; independent of the oracle)"""
    from scipy.spatial.transform import Rotation
    x, y, z, w = Rotation.from_matrix(R).as_quat()
    return np.array([w, x, y, z])


def _samples(x, y, J):
    """sample quaternions from the oracle's basis (numpy), half sphere q3 <= 0"""
    al = -np.pi + 2 * np.pi * np.arange(J) / J
    out = []
    for a, b in zip(x.astype(float), y.astype(float)):
        q1, q2 = oracle.alg1_basis(_unit(a), _unit(b))
        q = np.outer(np.cos(al / 2), q1) + np.outer(np.sin(al / 2), q2)
        q[q[:, 3] > 0] *= -1
        out.append(q)
    return np.array(out)


def test_noise_free_inlier_circles_pass_next_to_the_truth():
    pr = datagen.make_problem(60, 60, 0.0, 0.05, seed=3)
    for J in (36, 180):
        S = _samples(pr.x, pr.y, J)
        d = np.abs(S @ _quat(pr.R))            # |cos(angle)| between sample and +-q_true
        ang = np.arccos(np.clip(d.max(axis=1), -1, 1))
        assert ang.max() <= np.pi / (2 * J) + 1e-9


def test_bins_contain_their_samples_and_count_J_votes():
    rng = np.random.default_rng(4)
    pr = datagen.make_problem(40, 20, 0.01, 0.1, seed=5)
    x, y = pr.x.copy(), pr.y.copy()
    y[0] = -x[0]                               # antipodal row (a x b = 0)
    y[1] = x[1]                                # identical row
    for B, J in ((360, 180), (90, 37), (15, 8)):
        bins = oracle.alg1_bins(x, y, B, J)
        assert bins.shape == (40, J)
        S = _samples(x, y, J)
        p = S[..., :3] / (1.0 - S[..., 3:4])
        edges = np.linspace(-1, 1, B + 1)
        ijk = np.stack([bins // (B * B), (bins // B) % B, bins % B], -1)
        lo, hi = edges[ijk], edges[ijk + 1]
        tol = 1e-12
        inside = (p >= lo - tol) & ((p <= hi + tol) | (ijk == B - 1))
        assert inside.all()
        assert np.bincount(bins.ravel()).sum() == 40 * J


def test_alg1_solve_peaks_next_to_the_exact_winner():
    pr = datagen.cfg1()
    lin, votes, q = oracle.alg1_solve(pr.x, pr.y, 360, 180)
    ex = oracle.solve(pr.x, pr.y, pr.eps)
    B = 360
    ijk = np.array([lin // (B * B), (lin // B) % B, lin % B])
    assert np.abs(ijk - np.array(ex.cell)).max() <= 2
    # sampled votes <= samples that can reach one bin; > the outlier background
    assert 5 <= votes <= 180 * 50
    assert np.degrees(oracle.rotation_angle_between(q, _quat(pr.R))) < 2.0
