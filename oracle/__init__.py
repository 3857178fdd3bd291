"""ORACLE -- test infrastructure only.

ctypes wrapper around ``oracle/rv_oracle.cpp``, the plain single-threaded
double-precision CPU implementation of the rotation-voting definition (see the
header of rv_oracle.cpp for the definition and its citations into PAPER.md).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2506_11547_b200``) never imports it; the two share no
code.

Parity pins: every function is pinned by ``tests/test_oracle_pins.py`` against
closed forms, identities and worked examples the paper (or SPEC.md's worked
examples) fixes.  The search heuristic (child ordering) only changes cost and is
"parity unpinned" by nature; its result is pinned against the exhaustive scan.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rv_oracle.cpp")
_LIB = os.path.join(_HERE, "librvoracle.so")

DEFAULT_CHAIN = (5, 15, 45, 90, 180, 360)
GUARD = 1e-5


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (plain -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-ftree-vectorize", "-march=x86-64-v3",
               "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC", _SRC, "-o", _LIB + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class OrResult(C.Structure):
    _fields_ = [("q", C.c_double * 4), ("q_cell", C.c_double * 4), ("votes", C.c_uint32),
                ("n_inliers", C.c_uint32), ("cell", C.c_int32 * 3), ("flags", C.c_int32),
                ("B", C.c_int32), ("n_tied", C.c_int32), ("pair_evals", C.c_uint64),
                ("cells_evaluated", C.c_uint64), ("winner_near", C.c_uint32), ("pad", C.c_uint32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp, fp, u32p, u8p, i32p = (C.POINTER(C.c_double), C.POINTER(C.c_float),
                                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint8), C.POINTER(C.c_int32))
        L.or_quat_to_R.argtypes = [dp, dp]
        L.or_vote_stat.argtypes = [dp, dp, dp]; L.or_vote_stat.restype = C.c_double
        L.or_project.argtypes = [dp, dp]
        L.or_unproject.argtypes = [dp, dp]
        L.or_canonicalize.argtypes = [dp]
        L.or_constraint_M.argtypes = [dp, dp, dp]
        L.or_sym_eig4.argtypes = [dp, dp, dp]; L.or_sym_eig4.restype = C.c_int
        L.or_cell_center.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int64, dp]
        L.or_cell_is_candidate.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int64]
        L.or_cell_is_candidate.restype = C.c_int32
        L.or_cell_radius.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_int64]
        L.or_cell_radius.restype = C.c_double
        L.or_cell_bound_threshold.argtypes = [C.c_int32, C.c_int64, C.c_double]
        L.or_cell_bound_threshold.restype = C.c_double
        L.or_cell_quat.argtypes = [C.c_int32, C.c_int64, dp]
        L.or_candidates.argtypes = [C.c_int32, u32p, C.c_int64]; L.or_candidates.restype = C.c_int64
        L.or_normalize.argtypes = [fp, C.c_int64, dp]; L.or_normalize.restype = C.c_int64
        L.or_count_cells.argtypes = [fp, fp, C.c_int64, C.c_int32, u32p, C.c_int64, dp, C.c_double,
                                     u32p, u32p]
        L.or_count_cells.restype = C.c_int64
        L.or_pair_stats.argtypes = [fp, fp, C.c_int64, dp, dp]; L.or_pair_stats.restype = C.c_int64
        L.or_solve.argtypes = [fp, fp, C.c_int64, C.c_double, i32p, C.c_int32, C.c_int32, C.c_int32,
                               C.c_int32, C.c_double, C.POINTER(OrResult), u8p]
        L.or_solve.restype = C.c_int32
        L.or_refine.argtypes = [fp, fp, C.c_int64, C.c_double, dp, C.c_int32, dp, i32p, u8p]
        L.or_refine.restype = C.c_int32
        i64p = C.POINTER(C.c_int64)
        L.or_alg1_basis.argtypes = [dp, dp, dp, dp]
        L.or_alg1_bins.argtypes = [fp, fp, C.c_int64, C.c_int32, C.c_int32, i64p]
        L.or_alg1_bins.restype = C.c_int64
        L.or_alg1_solve.argtypes = [fp, fp, C.c_int64, C.c_int32, C.c_int32, i64p, u32p, dp]
        L.or_alg1_solve.restype = C.c_int64
        L.or_rigid_pairs.argtypes = [fp, fp, C.c_int64, C.c_double, C.c_int64, i64p, fp, fp]
        L.or_rigid_pairs.restype = C.c_int64
        L.or_translation_vote.argtypes = [fp, fp, C.c_int64, dp, C.c_double, C.c_double,
                                          C.c_double, i64p, u32p, dp, dp]
        L.or_translation_vote.restype = C.c_int64
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---- algebra ----------------------------------------------------------------

def quat_to_R(q) -> np.ndarray:
    q = _f64(q); R = np.zeros(9)
    lib().or_quat_to_R(_p(q, C.c_double), _p(R, C.c_double))
    return R.reshape(3, 3)


def vote_stat(q, a, b) -> float:
    q, a, b = _f64(q), _f64(a), _f64(b)
    return lib().or_vote_stat(_p(q, C.c_double), _p(a, C.c_double), _p(b, C.c_double))


def project(q) -> np.ndarray:
    q = _f64(q); p = np.zeros(3)
    lib().or_project(_p(q, C.c_double), _p(p, C.c_double))
    return p


def unproject(p) -> np.ndarray:
    p = _f64(p); q = np.zeros(4)
    lib().or_unproject(_p(p, C.c_double), _p(q, C.c_double))
    return q


def canonicalize(q) -> np.ndarray:
    q = _f64(q).copy()
    lib().or_canonicalize(_p(q, C.c_double))
    return q


def constraint_M(a, b) -> np.ndarray:
    a, b = _f64(a), _f64(b); M = np.zeros(16)
    lib().or_constraint_M(_p(a, C.c_double), _p(b, C.c_double), _p(M, C.c_double))
    return M.reshape(4, 4)


def sym_eig4(S):
    S = _f64(S).reshape(16); ev = np.zeros(4); V = np.zeros(16)
    lib().or_sym_eig4(_p(S, C.c_double), _p(ev, C.c_double), _p(V, C.c_double))
    return ev, V.reshape(4, 4)


# ---- grid ---------------------------------------------------------------------

def cell_center(B, i, j, k) -> np.ndarray:
    p = np.zeros(3)
    lib().or_cell_center(B, i, j, k, _p(p, C.c_double))
    return p


def cell_is_candidate(B, i, j, k) -> bool:
    return bool(lib().or_cell_is_candidate(B, i, j, k))


def cell_radius(B, i, j, k) -> float:
    return lib().or_cell_radius(B, i, j, k)


def cell_bound_threshold(B, lin, eps) -> float:
    return lib().or_cell_bound_threshold(B, int(lin), float(eps))


def cell_quat(B, lin) -> np.ndarray:
    q = np.zeros(4)
    lib().or_cell_quat(B, int(lin), _p(q, C.c_double))
    return q


def candidates(B) -> np.ndarray:
    m = lib().or_candidates(B, None, 0)
    out = np.zeros(m, np.uint32)
    lib().or_candidates(B, _p(out, C.c_uint32), m)
    return out


def lin_of(B, i, j, k) -> int:
    return (int(i) * B + int(j)) * B + int(k)


# ---- counting / solving -----------------------------------------------------------

def count_cells(x, y, B, lins, thr, band=GUARD):
    """(counts of s >= thr, counts of |s - thr| < band) per cell, exact double."""
    x, y = _f32(x), _f32(y)
    lins = np.ascontiguousarray(lins, np.uint32)
    thr = np.broadcast_to(np.asarray(thr, np.float64), lins.shape).copy()
    cnt = np.zeros(lins.size, np.uint32); nr = np.zeros(lins.size, np.uint32)
    bad = lib().or_count_cells(_p(x, C.c_float), _p(y, C.c_float), x.shape[0], B,
                               _p(lins, C.c_uint32), lins.size, _p(thr, C.c_double), band,
                               _p(cnt, C.c_uint32), _p(nr, C.c_uint32))
    if bad >= 0:
        raise ValueError(f"row {bad} cannot be normalised")
    return cnt, nr


def pair_stats(x, y, q) -> np.ndarray:
    x, y, q = _f32(x), _f32(y), _f64(q)
    s = np.zeros(x.shape[0])
    bad = lib().or_pair_stats(_p(x, C.c_float), _p(y, C.c_float), x.shape[0], _p(q, C.c_double),
                              _p(s, C.c_double))
    if bad >= 0:
        raise ValueError(f"row {bad} cannot be normalised")
    return s


@dataclass
class Solution:
    q: np.ndarray
    q_cell: np.ndarray
    votes: int
    n_inliers: int
    cell: tuple
    flags: int
    B: int
    n_tied: int
    pair_evals: int
    cells_evaluated: int
    winner_near: int
    mask: np.ndarray

    @property
    def lin(self) -> int:
        return lin_of(self.B, *self.cell)


def solve(x, y, eps, chain=DEFAULT_CHAIN, levels=0, exhaustive=False, refine_rounds=2,
          guard=GUARD) -> Solution:
    x, y = _f32(x), _f32(y)
    ch = np.ascontiguousarray(chain, np.int32)
    res = OrResult()
    mask = np.zeros(x.shape[0], np.uint8)
    rc = lib().or_solve(_p(x, C.c_float), _p(y, C.c_float), x.shape[0], float(eps),
                        _p(ch, C.c_int32), ch.size, int(levels), int(bool(exhaustive)),
                        int(refine_rounds), float(guard), C.byref(res), _p(mask, C.c_uint8))
    if rc == -1:
        raise ValueError("invalid arguments")
    if rc == -2:
        raise ValueError("a row cannot be normalised")
    return Solution(q=np.array(res.q[:]), q_cell=np.array(res.q_cell[:]), votes=res.votes,
                    n_inliers=res.n_inliers, cell=tuple(res.cell[:]), flags=res.flags, B=res.B,
                    n_tied=res.n_tied, pair_evals=res.pair_evals,
                    cells_evaluated=res.cells_evaluated, winner_near=res.winner_near,
                    mask=mask.astype(bool))


def refine(x, y, eps, q0, rounds=2):
    x, y, q0 = _f32(x), _f32(y), _f64(q0)
    q = np.zeros(4); fl = np.zeros(1, np.int32); mask = np.zeros(x.shape[0], np.uint8)
    rc = lib().or_refine(_p(x, C.c_float), _p(y, C.c_float), x.shape[0], float(eps),
                         _p(q0, C.c_double), rounds, _p(q, C.c_double), _p(fl, C.c_int32),
                         _p(mask, C.c_uint8))
    if rc != 0:
        raise ValueError("a row cannot be normalised")
    return q, int(fl[0]), mask.astype(bool)


def rotation_angle_between(qa, qb) -> float:
    """Geodesic rotation angle between two unit quaternions, stable near 0:
    4*asin(‖qa - s*qb‖/2) with s = sign(qa·qb) (SURVEY §8(c) parity rule 3).
    Plain definition; used by tests only."""
    qa, qb = np.asarray(qa, float), np.asarray(qb, float)
    s = 1.0 if float(qa @ qb) >= 0 else -1.0
    return float(4.0 * np.arcsin(min(1.0, np.linalg.norm(qa - s * qb) / 2.0)))


# ---- NEXT-4: the paper's Algorithm 1 ------------------------------

def alg1_basis(a, b):
    """(q_b1, q_b2) of the quaternion circle of a -> b (readings R13)."""
    a, b = _f64(a), _f64(b)
    q1, q2 = np.zeros(4), np.zeros(4)
    lib().or_alg1_basis(_p(a, C.c_double), _p(b, C.c_double), _p(q1, C.c_double),
                        _p(q2, C.c_double))
    return q1, q2


def alg1_bins(x, y, B=360, J=180) -> np.ndarray:
    """The accumulator bin (lin) of every sample, [n, J] int64."""
    x, y = _f32(x), _f32(y)
    n = x.shape[0]
    out = np.zeros((n, J), np.int64)
    rc = lib().or_alg1_bins(_p(x, C.c_float), _p(y, C.c_float), n, B, J, _p(out, C.c_int64))
    if rc != 0:
        raise ValueError(f"or_alg1_bins: {rc}")
    return out


def alg1_solve(x, y, B=360, J=180):
    """Algorithm 1 end to end: (lin of the max block, its votes, q of the block centre)."""
    x, y = _f32(x), _f32(y)
    lin = C.c_int64(); votes = C.c_uint32(); q = np.zeros(4)
    rc = lib().or_alg1_solve(_p(x, C.c_float), _p(y, C.c_float), x.shape[0], B, J,
                             C.byref(lin), C.byref(votes), _p(q, C.c_double))
    if rc != 0:
        raise ValueError(f"or_alg1_solve: {rc}")
    return lin.value, votes.value, q


# ---- NEXT-2: several rotations ------------------------------------

def solve_multi(x, y, eps, B, K, rho):
    """Top-K peaks with suppression, the plain definition (reading R16): exact counts of every
    candidate block of the B grid (s >= cos(eps), double), then greedily: peak 1 = the fullest
    block (ties -> lowest lin); peak k = the fullest block whose centre rotation is more than
    rho (rotation angle) from every earlier peak's centre -- |q_c . q_j| < cos(rho/2).  Returns
    a list of (lin, votes, n_tied, q_cell) with fewer than K entries when no block is left."""
    lins = candidates(B)
    cnt, _ = count_cells(x, y, B, lins, np.cos(eps))
    cnt = cnt.astype(np.int64)
    Q = np.array([cell_quat(B, int(l)) for l in lins])
    alive = np.ones(lins.size, bool)
    ch = np.cos(rho / 2.0)
    out = []
    for _ in range(K):
        if not alive.any():
            break
        c = np.where(alive, cnt, -1)
        best = c.max()
        tied = np.flatnonzero(c == best)
        e = tied[np.argmin(lins[tied])]
        q = Q[e].copy()
        canonicalize_q = q if q[3] <= 0 else -q
        out.append((int(lins[e]), int(best), int(tied.size), canonicalize_q))
        alive &= np.abs(Q @ Q[e]) < ch
    return out


# ---- NEXT-3: rigid pose front end ---------------------------------

def rigid_pairs(x, y, mu_t):
    """Kept pairs (i < j, lexicographic) of the length check: (ij [k,2], m [k,3], n [k,3])."""
    x, y = _f32(x), _f32(y)
    n = x.shape[0]
    k = lib().or_rigid_pairs(_p(x, C.c_float), _p(y, C.c_float), n, float(mu_t), 0, None,
                             None, None)
    ij = np.zeros((k, 2), np.int64)
    m = np.zeros((k, 3), np.float32)
    d = np.zeros((k, 3), np.float32)
    lib().or_rigid_pairs(_p(x, C.c_float), _p(y, C.c_float), n, float(mu_t), k,
                         _p(ij, C.c_int64), _p(m, C.c_float), _p(d, C.c_float))
    return ij, m, d


def translation_vote(x, y, q, lo=-5.0, hi=5.0, step=0.025):
    """(lin, votes, bin centre, mean of the bin's candidates) of the translation vote."""
    x, y, q = _f32(x), _f32(y), _f64(q)
    lin = C.c_int64(); votes = C.c_uint32(); t = np.zeros(3); tm = np.zeros(3)
    rc = lib().or_translation_vote(_p(x, C.c_float), _p(y, C.c_float), x.shape[0],
                                   _p(q, C.c_double), lo, hi, step, C.byref(lin),
                                   C.byref(votes), _p(t, C.c_double), _p(tm, C.c_double))
    if rc != 0:
        return None
    return lin.value, votes.value, t, tm
