"""Seeded synthetic correspondence generator shared by the oracle tests, the GPU
parity tests and bench.py.

This module holds NO arithmetic of the method (no quaternions, no R(q), no
vote statistic, no stereographic map): it only draws random 3-vectors and
rotation matrices.  Ground-truth rotations are drawn as Haar-random 3x3
matrices (QR of a Gaussian matrix with sign/determinant fix), so nothing here
depends on the paper's quaternion parameterisation.

Workload recipe (BASELINE.json ``configs``; stands in for the paper's
synthetic controlled experiments, §5.3.1, Table 1
lines 679-713 -- no dataset is used):

  x_i   : uniform on S^2 (normalised 3-d Gaussian).
  inlier: y_i = normalize(R x_i + N(0, sigma^2 I))   ("add a Gaussian
          perturbation ... and normalize all data again").
  outlier: y_i uniform on S^2, independent of x_i ("random mismatches").
  second structure (cfg3): inliers of an independent Haar R2.
  rows are randomly permuted; x, y are cast to float32 at the very end.

Random stream: numpy PCG64 via ``np.random.default_rng(seed)`` (batched
problem p uses ``default_rng([seed, p])``).  Draw order is fixed: R, (R2),
x, inlier noise, (structure-2 noise), outliers, permutation.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def haar_rotation(rng: np.random.Generator) -> np.ndarray:
    """Haar-distributed matrix on SO(3) (QR of a Gaussian, Mezzadri's sign fix)."""
    z = rng.standard_normal((3, 3))
    qm, rm = np.linalg.qr(z)
    qm = qm * np.sign(np.diag(rm))[None, :]
    if np.linalg.det(qm) < 0:
        qm[:, 0] = -qm[:, 0]
    return qm


def unit_vectors(rng: np.random.Generator, n: int) -> np.ndarray:
    v = rng.standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


@dataclass
class Problem:
    x: np.ndarray            # float32 [n,3]
    y: np.ndarray            # float32 [n,3]
    labels: np.ndarray       # uint8 [n]: 0 outlier, 1 inlier of R, 2 inlier of R2
    R: np.ndarray            # float64 [3,3] ground truth
    eps: float               # inlier angle (radians) used by the solve
    R2: np.ndarray | None = None
    sigma: float = 0.0
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.x.shape[0])


def make_problem(n: int, n_inl: int, sigma: float, eps: float, seed=0,
                 n_inl2: int = 0, sigma2: float = 0.0) -> Problem:
    """One rotation problem: n_inl inliers of R, n_inl2 of R2, rest outliers."""
    if n_inl + n_inl2 > n:
        raise ValueError("more inliers than correspondences")
    rng = np.random.default_rng(seed)
    R = haar_rotation(rng)
    R2 = haar_rotation(rng) if n_inl2 > 0 else None
    x = unit_vectors(rng, n)
    y = np.empty_like(x)
    lab = np.zeros(n, np.uint8)
    a = R @ x[:n_inl].T
    a = a.T + sigma * rng.standard_normal((n_inl, 3))
    y[:n_inl] = a / np.linalg.norm(a, axis=1, keepdims=True)
    lab[:n_inl] = 1
    if n_inl2:
        b = (R2 @ x[n_inl:n_inl + n_inl2].T).T + sigma2 * rng.standard_normal((n_inl2, 3))
        y[n_inl:n_inl + n_inl2] = b / np.linalg.norm(b, axis=1, keepdims=True)
        lab[n_inl:n_inl + n_inl2] = 2
    n_out = n - n_inl - n_inl2
    y[n_inl + n_inl2:] = unit_vectors(rng, n_out)
    perm = rng.permutation(n)
    return Problem(x=np.ascontiguousarray(x[perm], np.float32),
                   y=np.ascontiguousarray(y[perm], np.float32),
                   labels=lab[perm], R=R, R2=R2, eps=float(eps), sigma=float(sigma),
                   meta=dict(n=n, n_inl=n_inl, n_inl2=n_inl2, seed=seed))


# --- BASELINE.json configs -------------------------------------------------

def cfg1(seed=0) -> Problem:
    """N=100, 50 inliers sigma=0.01, 50 outliers, eps=0.05."""
    return make_problem(100, 50, 0.01, 0.05, seed)


def cfg2(seed=0) -> Problem:
    """N=1e4, 10% inliers sigma=0.01, eps=0.05."""
    return make_problem(10_000, 1_000, 0.01, 0.05, seed)


def cfg3(seed=0) -> Problem:
    """N=1e5, 5% inliers of R (sigma .02), 3% of R2 (sigma .02), 92% outliers, eps=.08."""
    return make_problem(100_000, 5_000, 0.02, 0.08, seed, n_inl2=3_000, sigma2=0.02)


def cfg4(seed=0) -> Problem:
    """N=1e6, 1% inliers sigma=0.01, 99% outliers, eps=0.05 (the metric's config)."""
    return make_problem(1_000_000, 10_000, 0.01, 0.05, seed)


@dataclass
class Batch:
    x: np.ndarray            # float32 [sum n_p, 3]
    y: np.ndarray
    offsets: np.ndarray      # int64 [P+1]
    eps: float
    problems: list


def cfg5(n_problems: int = 4096, n_per: int = 1000, seed=0) -> Batch:
    """4096 independent problems x N=1000, 80% outliers, sigma_p ~ U[0.005,0.03],
    eps = 3*sigma_max = 0.09 (sigma_max read as the range's upper bound)."""
    probs = []
    for p in range(n_problems):
        rng = np.random.default_rng([seed, p])
        sig = float(rng.uniform(0.005, 0.03))
        pr = make_problem(n_per, n_per // 5, sig, 0.09, seed=[seed, p, 1])
        probs.append(pr)
    return batch_of(probs, 0.09)


def batch_of(probs, eps: float) -> Batch:
    offs = np.zeros(len(probs) + 1, np.int64)
    offs[1:] = np.cumsum([p.n for p in probs])
    return Batch(x=np.ascontiguousarray(np.concatenate([p.x for p in probs])),
                 y=np.ascontiguousarray(np.concatenate([p.y for p in probs])),
                 offsets=offs, eps=eps, problems=probs)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}


# --- NEXT-3: rigid pose ----------------------------------------

@dataclass
class RigidProblem:
    x: np.ndarray        # [n, 3] fp32 points in [-1, 1]^3
    y: np.ndarray        # [n, 3] fp32: R x + t + delta N(0, I) for inliers
    labels: np.ndarray   # 1 inlier, 0 outlier
    R: np.ndarray
    t: np.ndarray
    delta: float
    meta: dict


def make_rigid(n: int, outlier_ratio: float, delta: float, seed=0) -> RigidProblem:
    """The paper's synthetic rigid-motion setting: R Haar, t uniform in [-1,1]^3,
    x uniform in [-1,1]^3, y = R x + t + delta N(0, I); outliers: x and y independent uniform
    in [-1,1]^3; rows permuted."""
    rng = np.random.default_rng(seed)
    R = haar_rotation(rng)
    t = rng.uniform(-1.0, 1.0, 3)
    n_out = int(round(outlier_ratio * n))
    n_in = n - n_out
    x = rng.uniform(-1.0, 1.0, (n, 3))
    y = np.empty_like(x)
    y[:n_in] = x[:n_in] @ R.T + t + delta * rng.standard_normal((n_in, 3))
    y[n_in:] = rng.uniform(-1.0, 1.0, (n_out, 3))
    lab = np.zeros(n, np.uint8)
    lab[:n_in] = 1
    perm = rng.permutation(n)
    return RigidProblem(x=np.ascontiguousarray(x[perm], np.float32),
                        y=np.ascontiguousarray(y[perm], np.float32), labels=lab[perm], R=R,
                        t=t, delta=float(delta),
                        meta=dict(n=n, outlier_ratio=outlier_ratio, seed=seed))
