"""Pins of the CPU oracle (oracle/rv_oracle.cpp) against what the paper and the
mathematics fix -- never against the oracle itself.

Each test names the passage it pins.  Independent references used here:
scipy's Rotation (a library rotation routine), numpy's eigh/SVD, hand-evaluated
worked examples (SPEC.md, tagged [TRIVIAL]/[DERIVED]), closed forms from the
paper (quaternion circle P:282-296, Appendix A/D/E), brute force on tiny grids.
"""
import itertools
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation as Rot

import datagen

S2 = math.sqrt(2.0) / 2.0


def scipy_R(q):
    return Rot.from_quat(np.asarray(q, float), scalar_first=True).as_matrix()


def rand_quat(rng):
    q = rng.standard_normal(4)
    return q / np.linalg.norm(q)


# ---- R(q): P:955-961 ----------------------------------------------------------------

def test_quat_to_R_worked_examples(oracle_mod):
    o = oracle_mod
    # S:65-67 (quat_to_matrix examples)
    assert np.allclose(o.quat_to_R([1, 0, 0, 0]), np.eye(3), atol=1e-15)
    R = o.quat_to_R([S2, 0, 0, S2])
    assert np.allclose(R @ [1, 0, 0], [0, 1, 0], atol=1e-15)
    assert np.allclose(o.quat_to_R([0, 1, 0, 0]), np.diag([1, -1, -1]), atol=1e-15)
    # 90 deg about x sends y -> z; about y sends z -> x  (right-hand rule)
    assert np.allclose(o.quat_to_R([S2, S2, 0, 0]) @ [0, 1, 0], [0, 0, 1], atol=1e-15)
    assert np.allclose(o.quat_to_R([S2, 0, S2, 0]) @ [0, 0, 1], [1, 0, 0], atol=1e-15)


def test_quat_to_R_matches_library(oracle_mod):
    rng = np.random.default_rng(1)
    for _ in range(200):
        q = rand_quat(rng)
        R = oracle_mod.quat_to_R(q)
        assert np.allclose(R, scipy_R(q), atol=1e-14)
        assert np.allclose(R, oracle_mod.quat_to_R(-q), atol=1e-15)  # q == -q
        assert abs(np.linalg.det(R) - 1) < 1e-13


# ---- vote statistic and the Appendix-A matrix M -------------------------

def test_vote_stat_is_bRa_and_quadratic_form(oracle_mod):
    o = oracle_mod
    rng = np.random.default_rng(2)
    for _ in range(200):
        q = rand_quat(rng)
        a = datagen.unit_vectors(rng, 1)[0]
        b = datagen.unit_vectors(rng, 1)[0]
        s = o.vote_stat(q, a, b)
        assert abs(s - b @ scipy_R(q) @ a) < 1e-14
        M = o.constraint_M(a, b)
        assert np.allclose(M, M.T, atol=1e-15)                   # symmetric
        assert abs(q @ M @ q - s) < 1e-14                        # qᵀMq = bᵀRa
        ev = np.linalg.eigvalsh(M)
        assert np.allclose(ev, [-1, -1, 1, 1], atol=1e-13)       # (λ²-1)² = 0
        assert np.allclose(M @ M, np.eye(4), atol=1e-13)
        assert abs(np.trace(M)) < 1e-14


def test_constraint_satisfied_iff_rotation_maps(oracle_mod):
    """R a = b  <=>  bᵀRa = 1."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        q = rand_quat(rng)
        a = datagen.unit_vectors(rng, 1)[0]
        b = scipy_R(q) @ a
        assert abs(oracle_mod.vote_stat(q, a, b) - 1.0) < 1e-14
        q2 = q + 0.01 * rng.standard_normal(4)
        q2 /= np.linalg.norm(q2)
        ang = np.arccos(np.clip(b @ scipy_R(q2) @ a, -1, 1))
        assert abs(oracle_mod.vote_stat(q2, a, b) - math.cos(ang)) < 1e-13


def quaternion_circle_basis(a, b):
    """q_b1, q_b2 exactly as P:246-296: q_b1 = minimal geodesic rotation a->b
    (P:248-251), q_b2 = [-bᵀq123, q0 b + b x q123]."""
    theta = math.acos(np.clip(a @ b, -1, 1))
    c = np.cross(a, b)
    c /= np.linalg.norm(c)
    qb1 = np.concatenate([[math.cos(theta / 2)], math.sin(theta / 2) * c])
    q0, q123 = qb1[0], qb1[1:]
    qb2 = np.concatenate([[-(b @ q123)], q0 * b + np.cross(b, q123)])
    return qb1, qb2


def test_quaternion_circle_passes_constraint(oracle_mod):
    """Every q(α) = q_b1 cos(α/2) + q_b2 sin(α/2) satisfies R a = b and
    lies in the +1 eigenspace of M."""
    o = oracle_mod
    rng = np.random.default_rng(4)
    for _ in range(50):
        a, b = datagen.unit_vectors(rng, 2)
        qb1, qb2 = quaternion_circle_basis(a, b)
        assert abs(qb1 @ qb2) < 1e-14 and abs(qb2 @ qb2 - 1) < 1e-14
        M = o.constraint_M(a, b)
        for al in np.linspace(-math.pi, math.pi, 37):
            q = qb1 * math.cos(al / 2) + qb2 * math.sin(al / 2)
            assert abs(o.vote_stat(q, a, b) - 1.0) < 1e-13
            assert np.allclose(M @ q, q, atol=1e-13)


def test_appendix_D_rows(oracle_mod):
    """[[0,(a-b)ᵀ],[-(a-b),[a+b]x]] q = 0 for R a = b; its columns are
    -1 eigenvectors of M."""
    o = oracle_mod
    rng = np.random.default_rng(5)
    for _ in range(50):
        q = rand_quat(rng)
        a = datagen.unit_vectors(rng, 1)[0]
        b = scipy_R(q) @ a
        d, s = a - b, a + b
        sx = np.array([[0, -s[2], s[1]], [s[2], 0, -s[0]], [-s[1], s[0], 0]])
        D = np.zeros((4, 4))
        D[0, 1:] = d
        D[1:, 0] = -d
        D[1:, 1:] = sx
        assert np.allclose(D @ q, 0, atol=1e-14)
        M = o.constraint_M(a, b)
        E = np.zeros((4, 4))
        E[0, 1:] = -d
        E[1:, 0] = -d
        E[1:, 1:] = sx.T
        assert np.allclose(M @ E, -E, atol=1e-13)


# ---- stereographic map and hemisphere ------------------------------

def test_stereographic_examples(oracle_mod):
    o = oracle_mod
    assert np.allclose(o.project([1, 0, 0, 0]), [1, 0, 0])
    assert np.allclose(o.project([0, 0, 0, -1]), [0, 0, 0])
    assert np.allclose(o.project([-S2, 0, 0, -S2]), [-(math.sqrt(2) - 1), 0, 0])
    assert np.allclose(o.unproject([0, 0, 0]), [0, 0, 0, -1])
    assert np.allclose(o.unproject([1, 0, 0]), [1, 0, 0, 0])
    rng = np.random.default_rng(6)
    for _ in range(1000):
        p = rng.uniform(-1, 1, 3)
        q = o.unproject(p)
        assert abs(np.linalg.norm(q) - 1) < 1e-15
        assert np.allclose(o.project(q), p, atol=1e-14)
        assert (q[3] <= 0) == (p @ p <= 1)  # the ball is the q3 <= 0 hemisphere


def test_canonicalize_examples(oracle_mod):
    o = oracle_mod
    assert np.allclose(o.canonicalize([S2, 0, 0, S2]), [-S2, 0, 0, -S2])
    assert np.allclose(o.canonicalize([1, 0, 0, 0]), [1, 0, 0, 0])
    assert np.allclose(o.canonicalize([-1, 0, 0, 0]), [1, 0, 0, 0])
    assert np.allclose(o.canonicalize([0, -1, 0, 0]), [0, 1, 0, 0])


# ---- Jacobi eigen-solver vs library ------------------------------------------------------

def test_sym_eig4_matches_numpy(oracle_mod):
    rng = np.random.default_rng(7)
    for _ in range(300):
        A = rng.standard_normal((4, 4))
        S = A + A.T
        ev, V = oracle_mod.sym_eig4(S)
        w, U = np.linalg.eigh(S)
        assert np.allclose(ev, w[::-1], atol=1e-12)
        for j in range(4):
            assert abs(abs(V[:, j] @ U[:, 3 - j]) - 1) < 1e-10
        assert np.allclose(V @ np.diag(ev) @ V.T, S, atol=1e-12)


# ---- the grid -----------------------------------------------------------------------

@pytest.mark.parametrize("B", [1, 2, 5, 15, 16, 45])
def test_candidate_cells_brute_force(oracle_mod, B):
    """candidate <=> the block meets the closed unit ball; checked by clamping the
    origin onto the box in numpy (independent float computation)."""
    idx = np.arange(B)
    lo = -1 + 2 * idx / B
    hi = lo + 2 / B
    closest = np.clip(0.0, lo, hi)
    d2 = (closest[:, None, None] ** 2 + closest[None, :, None] ** 2 + closest[None, None, :] ** 2)
    expect = np.flatnonzero(d2.reshape(-1) <= 1 + 1e-12).astype(np.uint32)
    got = oracle_mod.candidates(B)
    assert np.array_equal(got, expect)
    if B == 15:
        assert got.size == 2295
    if B == 45:
        assert got.size == 52461


@pytest.mark.parametrize("B", [1, 2, 5, 15, 45, 360])
def test_cell_center_is_block_midpoint(oracle_mod, B):
    """P:488 divides [-1,1]^3 into B blocks per axis; P:502 returns "the center of the
    block".  The centre of block i along an axis is the midpoint of the i-th interval of
    np.linspace(-1, 1, B + 1) (an independent construction of the same grid).  A
    corner-for-centre mistake (p = -1 + 2i/B) fails this by 1/B."""
    edges = np.linspace(-1.0, 1.0, B + 1)
    mids = 0.5 * (edges[:-1] + edges[1:])
    rng = np.random.default_rng(B)
    idx = [(0, 0, 0), (B - 1, B - 1, B - 1)] + [tuple(rng.integers(0, B, 3)) for _ in range(40)]
    for i, j, k in idx:
        p = oracle_mod.cell_center(B, int(i), int(j), int(k))
        assert np.allclose(p, [mids[i], mids[j], mids[k]], rtol=0, atol=4e-16), (B, i, j, k)
        # the centre lies strictly inside its block, half a step from both faces
        for a, v in enumerate((i, j, k)):
            assert edges[v] < p[a] < edges[v + 1]
            assert abs((p[a] - edges[v]) - (edges[v + 1] - p[a])) < 1e-15


def test_cell_quat_hand_evaluated(oracle_mod):
    """q_c = P'(p_c): P'(p) = [2p/(1+p.p), (p.p-1)/(1+p.p)].  Values worked out by
    hand as exact fractions at block centres (no code shared with the oracle):
      B=1 (0,0,0):  p = 0                   -> q = (0, 0, 0, -1)
      B=2 (1,1,1):  p = (1/2, 1/2, 1/2)     -> p.p = 3/4,  q = (4/7, 4/7, 4/7, -1/7)
      B=2 (0,1,1):  p = (-1/2, 1/2, 1/2)    -> q = (-4/7, 4/7, 4/7, -1/7)
      B=4 (3,0,1):  p = (3/4, -3/4, -1/4)   -> p.p = 19/16, q = (24/35, -24/35, -8/35, 3/35)
                    (centre outside the ball: q3 > 0, the same rotation as -q, R4)
      B=5 (2,2,4):  p = (0, 0, 4/5)         -> p.p = 16/25, q = (0, 0, 40/41, -9/41)
    A corner-for-centre or a sign/ordering mistake (pole, scalar-first) fails here."""
    o = oracle_mod
    cases = [
        (1, (0, 0, 0), (0, 0, 0, -1)),
        (2, (1, 1, 1), (4 / 7, 4 / 7, 4 / 7, -1 / 7)),
        (2, (0, 1, 1), (-4 / 7, 4 / 7, 4 / 7, -1 / 7)),
        (4, (3, 0, 1), (24 / 35, -24 / 35, -8 / 35, 3 / 35)),
        (5, (2, 2, 4), (0, 0, 40 / 41, -9 / 41)),
    ]
    for B, (i, j, k), q in cases:
        got = o.cell_quat(B, o.lin_of(B, i, j, k))
        assert np.allclose(got, q, rtol=0, atol=1e-15), (B, i, j, k, got)
        assert abs(np.linalg.norm(got) - 1) < 1e-15


def test_count_cells_near_band_independent(oracle_mod):
    """or_count_cells' second output is #{i : |s_i(q_c) - t| < band}, the band the GPU
    parity tests accept (SURVEY §8(c) parity rule).  Recomputed here in numpy from
    scipy's rotation of the block quaternion: near = #{s > t - band} - #{s >= t + band},
    and the count = #{s >= t}.  Bands of 1e-2 / 3e-3 / 1e-5 so both are non-trivial;
    a widened or narrowed band, or a one-sided band, fails."""
    o = oracle_mod
    pr = datagen.make_problem(4000, 400, 0.01, 0.05, seed=21)
    xn = pr.x.astype(np.float64)
    yn = pr.y.astype(np.float64)
    xn /= np.linalg.norm(xn, axis=1, keepdims=True)
    yn /= np.linalg.norm(yn, axis=1, keepdims=True)
    rng = np.random.default_rng(22)
    B = 45
    lins = np.sort(rng.choice(o.candidates(B), 24, replace=False)).astype(np.uint32)
    total_near = 0
    for band in (1e-2, 3e-3, 1e-5):
        t = rng.uniform(0.2, 0.99, lins.size)
        cnt, near = o.count_cells(pr.x, pr.y, B, lins, t, band=band)
        for m, lin in enumerate(lins):
            q = o.cell_quat(B, int(lin))
            s = np.einsum("ij,ij->i", yn, xn @ scipy_R(q).T)
            # pairs within 1e-12 of an edge could round either way: skip the cell then
            edge = np.abs(np.abs(s - t[m]) - band) < 1e-12
            if edge.any() or (np.abs(s - t[m]) < 1e-12).any():
                continue
            assert near[m] == int((s > t[m] - band).sum() - (s >= t[m] + band).sum())
            assert cnt[m] == int((s >= t[m]).sum())
            total_near += int(near[m])
    assert total_near > 100  # the band is exercised


def test_cell_radius_bounds_rotation_spread(oracle_mod):
    """For any p in a block, angle(R(P'(p)), R(P'(p_c))) <= r(c) (R6).
    Also checks the bound is not vacuous: the corner nearest the origin reaches
    at least a third of it."""
    o = oracle_mod
    rng = np.random.default_rng(8)
    for B in (3, 5, 15, 45):
        cells = o.candidates(B)
        for lin in rng.choice(cells, size=min(60, cells.size), replace=False):
            i, j, k = lin // (B * B), (lin // B) % B, lin % B
            pc = o.cell_center(B, i, j, k)
            Rc = scipy_R(o.unproject(pc))
            r = o.cell_radius(B, i, j, k)
            worst = 0.0
            corners = [pc + np.array(s) / B for s in itertools.product((-1, 1), repeat=3)]
            pts = [pc + rng.uniform(-1, 1, 3) / B for _ in range(40)] + corners
            for p in pts:
                ang = Rot.from_matrix(Rc.T @ scipy_R(o.unproject(p))).magnitude()
                worst = max(worst, ang)
                assert ang <= r * (1 + 1e-12)
            assert worst >= r / 3


def test_bound_dominates_descendants(oracle_mod):
    """UB(c) = #{s(q_c) >= cos(min(pi, eps + r(c)))} >= count of every finer block
    whose centre lies in c (brute force over all descendants)."""
    o = oracle_mod
    rng = np.random.default_rng(9)
    for trial in range(6):
        n = 40
        pr = datagen.make_problem(n, 20, 0.02, 0.1, seed=100 + trial)
        Bc, Bf = 5, 20
        cells = o.candidates(Bc)
        f = Bf // Bc
        for lin in rng.choice(cells, 20, replace=False):
            t = o.cell_bound_threshold(Bc, lin, pr.eps)
            ub, _ = o.count_cells(pr.x, pr.y, Bc, [lin], t, band=0)
            i, j, k = lin // (Bc * Bc), (lin // Bc) % Bc, lin % Bc
            kids = [o.lin_of(Bf, f * i + a, f * j + b, f * k + c)
                    for a in range(f) for b in range(f) for c in range(f)]
            cnt, _ = o.count_cells(pr.x, pr.y, Bf, kids, math.cos(pr.eps), band=0)
            assert ub[0] >= cnt.max()


# ---- two correspondences, incompatibility (App. E) ----------------------

def test_two_correspondences_closed_form(oracle_mod):
    """Noise-free pair: the two great circles meet at ±q: λmax of
    M1+M2 is 2 and simple, its eigenvector is ±q_true; the full solve on N=2
    returns it.  R = 90° about z maps fp32 inputs exactly."""
    o = oracle_mod
    q_true = np.array([S2, 0, 0, S2])
    R = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    assert np.allclose(R, scipy_R(q_true), atol=1e-15)
    x = np.array([[0.25, -0.5, 0.75], [0.5, 0.125, -0.625]], np.float32)
    y = (R @ x.astype(float).T).T.astype(np.float32)
    assert np.array_equal((R @ x.astype(float).T).T, y.astype(float))  # exact in fp32
    xn = x.astype(float) / np.linalg.norm(x.astype(float), axis=1, keepdims=True)
    yn = y.astype(float) / np.linalg.norm(y.astype(float), axis=1, keepdims=True)
    S = o.constraint_M(xn[0], yn[0]) + o.constraint_M(xn[1], yn[1])
    ev, V = o.sym_eig4(S)
    assert abs(ev[0] - 2) < 1e-13 and ev[1] < 2 - 1e-3
    assert abs(abs(V[:, 0] @ q_true) - 1) < 1e-13
    sol = o.solve(x, y, eps=0.05, chain=(5, 15, 45), levels=3)
    assert sol.votes == 2 and sol.flags & 1
    assert o.rotation_angle_between(sol.q, q_true) < 1e-9
    # generic rotation: fp32 rounding of y limits agreement to ~1e-7 rad
    rng = np.random.default_rng(10)
    for _ in range(10):
        qt = o.canonicalize(rand_quat(rng))
        x = datagen.unit_vectors(rng, 2).astype(np.float32)
        y = (scipy_R(qt) @ x.astype(float).T).T.astype(np.float32)
        sol = o.solve(x, y, eps=0.05)      # 360³ grid: cell spread <= 0.02 rad
        assert sol.votes == 2
        assert o.rotation_angle_between(sol.q, qt) < 1e-5


def test_incompatible_pair(oracle_mod):
    """App. E: two pairs rotated about one axis r by different angles admit no common
    rotation -> λmax(M1+M2) < 2; same angle -> = 2."""
    o = oracle_mod
    rng = np.random.default_rng(11)
    for _ in range(20):
        r = datagen.unit_vectors(rng, 1)[0]
        x1, x2 = datagen.unit_vectors(rng, 2)
        al, be = np.radians(20), np.radians(60)
        y1 = Rot.from_rotvec(al * r).apply(x1)
        y2 = Rot.from_rotvec(be * r).apply(x2)
        S = o.constraint_M(x1, y1) + o.constraint_M(x2, y2)
        assert o.sym_eig4(S)[0][0] < 2 - 1e-6
        y2c = Rot.from_rotvec(al * r).apply(x2)
        S = o.constraint_M(x1, y1) + o.constraint_M(x2, y2c)
        assert abs(o.sym_eig4(S)[0][0] - 2) < 1e-12


# ---- refinement = Horn = SVD ----------------------------------

def umeyama_R(xs, ys):
    """SVD solution R* = U diag(1,1,det(UVᵀ)) Vᵀ of B = Σ y xᵀ."""
    Bm = ys.T @ xs
    U, _, Vt = np.linalg.svd(Bm)
    D = np.diag([1, 1, np.linalg.det(U @ Vt)])
    return U @ D @ Vt


def test_refinement_equals_svd(oracle_mod):
    o = oracle_mod
    for seed in range(5):
        pr = datagen.make_problem(2000, 600, 0.02, 0.08, seed=seed)
        q0 = Rot.from_matrix(pr.R).as_quat(scalar_first=True)
        q0 = q0 + 0.002 * np.random.default_rng(seed).standard_normal(4)
        q0 /= np.linalg.norm(q0)
        q1, fl, _ = o.refine(pr.x, pr.y, pr.eps, q0, rounds=1)
        assert fl == 1
        xn = pr.x.astype(float); xn /= np.linalg.norm(xn, axis=1, keepdims=True)
        yn = pr.y.astype(float); yn /= np.linalg.norm(yn, axis=1, keepdims=True)
        s = np.einsum("ni,ij,nj->n", yn, scipy_R(q0), xn)      # inlier set at q0 (numpy)
        I = s >= math.cos(pr.eps)
        Rs = umeyama_R(xn[I], yn[I])
        ang = Rot.from_matrix(Rs.T @ scipy_R(q1)).magnitude()
        assert ang < 1e-9


def test_noise_free_outlier_free_exact(oracle_mod):
    o = oracle_mod
    pr = datagen.make_problem(500, 500, 0.0, 0.01, seed=3)
    sol = o.solve(pr.x, pr.y, pr.eps, chain=(15, 45, 90, 180, 360), levels=5)
    assert sol.n_inliers == 500 and sol.votes >= 1
    xn = pr.x.astype(float); xn /= np.linalg.norm(xn, axis=1, keepdims=True)
    yn = pr.y.astype(float); yn /= np.linalg.norm(yn, axis=1, keepdims=True)
    ang = Rot.from_matrix(umeyama_R(xn, yn).T @ o.quat_to_R(sol.q)).magnitude()
    assert ang < 1e-9
    assert Rot.from_matrix(pr.R.T @ o.quat_to_R(sol.q)).magnitude() < 1e-6  # fp32 inputs


# ---- statistics of the vote ---------------------------------------------------------------

def test_background_counts_are_binomial(oracle_mod):
    """y uniform on S² independent of x => s uniform on [-1,1] (Archimedes), so a
    pure-outlier count is Binomial(n, (1-t)/2)."""
    o = oracle_mod
    n = 20000
    pr = datagen.make_problem(n, 0, 0.0, 0.3, seed=12)
    B = 15
    cells = o.candidates(B)[::23]
    t = math.cos(0.3)
    cnt, _ = o.count_cells(pr.x, pr.y, B, cells, t, band=0)
    p = (1 - t) / 2
    z = (cnt.mean() - n * p) / math.sqrt(n * p * (1 - p) / cells.size)
    assert abs(z) < 4
    assert cnt.std() < 2 * math.sqrt(n * p * (1 - p))


def test_inlier_count_at_truth(oracle_mod):
    """Every noise-free inlier circle passes through q_true: at q_true every
    inlier has s = 1 up to fp32 rounding of the inputs."""
    o = oracle_mod
    pr = datagen.make_problem(1000, 300, 0.0, 0.05, seed=13)
    qt = Rot.from_matrix(pr.R).as_quat(scalar_first=True)
    s = o.pair_stats(pr.x, pr.y, qt)
    assert np.all(np.abs(s[pr.labels == 1] - 1) < 1e-6)


# ---- certified search == exhaustive scan (the definition) ------------------------------------

CHAINS = [(3, 9, 27), (5, 15, 45), (4, 8, 16, 32), (2, 4, 8, 16), (6, 18), (5, 10, 20, 40)]


def _random_problem(rng):
    n = int(rng.integers(2, 61))
    kind = rng.integers(0, 4)
    eps = float(rng.choice([0.02, 0.05, 0.1, 0.3, 1.0, 2.5]))
    n_in = int(rng.integers(0, n + 1))
    sigma = float(rng.choice([0.0, 0.01, 0.05]))
    pr = datagen.make_problem(n, n_in, sigma, eps, seed=int(rng.integers(1 << 30)))
    x, y = pr.x.copy(), pr.y.copy()
    if kind == 1:          # y = x rows (identity-compatible)
        y[: n // 3] = x[: n // 3]
    elif kind == 2:        # y = -x rows (antipodal, the minimal-geodesic singular case)
        y[: n // 3] = -x[: n // 3]
    elif kind == 3 and n >= 6:   # second structure
        pr2 = datagen.make_problem(n // 2, n // 2, sigma, eps, seed=int(rng.integers(1 << 30)))
        x[: n // 2], y[: n // 2] = pr2.x, pr2.y
    return x, y, eps


def test_certified_equals_exhaustive_random(oracle_mod):
    o = oracle_mod
    rng = np.random.default_rng(14)
    checked = 0
    for trial in range(400):
        x, y, eps = _random_problem(rng)
        chain = CHAINS[trial % len(CHAINS)]
        ex = o.solve(x, y, eps, chain=chain, levels=len(chain), exhaustive=True)
        for L in range(2, len(chain) + 1):
            ce = o.solve(x, y, eps, chain=chain, levels=L)
            assert (ce.cell, ce.votes, ce.n_tied) == (ex.cell, ex.votes, ex.n_tied), (trial, chain, L)
            assert np.allclose(ce.q, ex.q, atol=1e-15)
            checked += 1
    assert checked > 400


def test_certified_equals_exhaustive_cfg1_fine_grid(oracle_mod):
    """BASELINE config 1 on the paper's 360³ grid (ε = 1/180)."""
    o = oracle_mod
    pr = datagen.cfg1()
    ex = o.solve(pr.x, pr.y, pr.eps, exhaustive=True)
    for L in (2, 3, 5, 6):
        ce = o.solve(pr.x, pr.y, pr.eps, levels=L)
        assert (ce.cell, ce.votes, ce.n_tied) == (ex.cell, ex.votes, ex.n_tied)
    assert ex.votes >= 45
    ang = Rot.from_matrix(pr.R.T @ o.quat_to_R(ex.q)).magnitude()
    assert np.degrees(ang) < 1.0      # success criterion e_R <= 5 deg


def test_solve_recovers_rotation_high_outliers(oracle_mod):
    """99% outliers, N=2e4: e_R far below the paper's 5° success bar."""
    o = oracle_mod
    pr = datagen.make_problem(20000, 200, 0.01, 0.05, seed=15)
    sol = o.solve(pr.x, pr.y, pr.eps)
    ang = np.degrees(Rot.from_matrix(pr.R.T @ o.quat_to_R(sol.q)).magnitude())
    assert ang < 0.5
    assert sol.votes >= 190
    assert sol.flags == 1


def test_degenerate_flags(oracle_mod):
    o = oracle_mod
    rng = np.random.default_rng(16)
    x = datagen.unit_vectors(rng, 3).astype(np.float32)
    y = datagen.unit_vectors(rng, 3).astype(np.float32)
    sol = o.solve(x, y, 0.001, chain=(5, 15, 45), levels=3)
    if sol.votes < 2:
        assert sol.flags & 2
    with pytest.raises(ValueError):
        o.solve(x[:1], y[:1], 0.05)
    bad = x.copy(); bad[1] = 0
    with pytest.raises(ValueError):
        o.solve(bad, y, 0.05)


def test_rotation_angle_stable_form(oracle_mod):
    """4·asin(‖qa − s·qb‖/2) equals e_R = arccos((tr(RaᵀRb) − 1)/2)."""
    o = oracle_mod
    rng = np.random.default_rng(17)
    for _ in range(100):
        qa, qb = rand_quat(rng), rand_quat(rng)
        tr = np.trace(scipy_R(qa).T @ scipy_R(qb))
        eR = math.acos(np.clip((tr - 1) / 2, -1, 1))
        assert abs(o.rotation_angle_between(qa, qb) - eR) < 1e-7
