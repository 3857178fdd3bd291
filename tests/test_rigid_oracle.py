"""Pins of the oracle's rigid-pose front end (NEXT-3):
* pairs: the kept set equals an independent numpy brute force of the length check
  |‖x_i - x_j‖ - ‖y_i - y_j‖| <= mu_t over all i < j, in lexicographic order; every inlier pair
  of a noise-free rigid scene is kept at mu_t = 0 up to rounding (R x + t preserves lengths);
* the translation vote: for a noise-free scene and the true rotation every inlier's candidate
  t_i equals t, so the winning bin contains t and holds every inlier; the mean is t;
* end to end on the paper's synthetic setting, the oracle's rotation of the pairs
  and its translation land within the grid's resolution of the truth."""
import numpy as np
import pytest

import datagen
import oracle


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def _quat(R):
    from scipy.spatial.transform import Rotation
    x, y, z, w = Rotation.from_matrix(R).as_quat()
    return np.array([w, x, y, z])


def test_pairs_equal_brute_force():
    p = datagen.make_rigid(120, 0.7, 0.01, seed=3)
    for mu in (0.0, 0.01, 0.05, 0.3):
        ij, m, d = oracle.rigid_pairs(p.x, p.y, mu)
        X, Y = p.x.astype(np.float64), p.y.astype(np.float64)
        i, j = np.triu_indices(len(X), 1)
        lm = np.linalg.norm(X[i] - X[j], axis=1)
        ld = np.linalg.norm(Y[i] - Y[j], axis=1)
        keep = np.abs(lm - ld) <= mu
        # rows where the length difference is within 1e-12 of mu may round either way
        amb = np.abs(np.abs(lm - ld) - mu) < 1e-12
        ref = set(zip(i[keep & ~amb], j[keep & ~amb]))
        got = set(map(tuple, ij))
        assert ref <= got and got - ref <= set(zip(i[amb], j[amb]))
        assert np.all(np.diff(ij[:, 0] * 1000 + ij[:, 1]) > 0)          # pair order
        k = ij[:, 0], ij[:, 1]
        assert np.allclose(m, (X[k[0]] - X[k[1]]).astype(np.float32))
        assert np.allclose(d, (Y[k[0]] - Y[k[1]]).astype(np.float32))


def test_noise_free_inlier_pairs_survive_a_tight_check():
    p = datagen.make_rigid(80, 0.5, 0.0, seed=4)
    ij, _, _ = oracle.rigid_pairs(p.x, p.y, 1e-5)
    inl = set(np.flatnonzero(p.labels == 1))
    kept = {(a, b) for a, b in ij}
    assert {(a, b) for a in inl for b in inl if a < b} <= kept


def test_translation_vote_noise_free():
    p = datagen.make_rigid(200, 0.6, 0.0, seed=5)
    lin, votes, t, tm = oracle.translation_vote(p.x, p.y, _quat(p.R))
    assert votes >= int((p.labels == 1).sum())
    assert np.all(np.abs(t - p.t) <= 0.0125 + 1e-9)
    assert np.allclose(tm, p.t, atol=1e-6)


def test_rigid_end_to_end_oracle():
    from scipy.spatial.transform import Rotation as Rot
    p = datagen.make_rigid(300, 0.8, 0.01, seed=6)
    ij, m, d = oracle.rigid_pairs(p.x, p.y, 0.05)
    sol = oracle.solve(m, d, 0.05)
    w, a, b, c = sol.q
    err = np.degrees((Rot.from_matrix(p.R).inv() * Rot.from_quat([a, b, c, w])).magnitude())
    assert err < 1.0
    lin, votes, t, tm = oracle.translation_vote(p.x, p.y, sol.q)
    assert np.linalg.norm(tm - p.t) < 0.05
