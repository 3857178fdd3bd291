"""Test helper: drive the library's host planner with counts from the CPU oracle."""
import math

import numpy as np

import oracle
from paper_2506_11547_b200 import rotvote as rvmod

GUARD = 1e-5


def oracle_counts(x, y, eps, B, mode, lins, guard=GUARD):
    """Counts of the request in `mode`, computed exactly (double) by the oracle with the
    oracle's own bound threshold (rotvote.h RV_MODE_* semantics, exact arithmetic)."""
    lins = np.asarray(lins, np.uint32)
    if lins.size == 0:
        z = np.zeros(0, np.uint32)
        return z, z
    tau = math.cos(eps)
    if mode == rvmod.RV_MODE_BOUND:
        thr = np.array([oracle.cell_bound_threshold(B, int(l), eps) for l in lins]) - guard
        a, _ = oracle.count_cells(x, y, B, lins, thr, band=0)
        return a, None
    if mode == rvmod.RV_MODE_FINAL:
        a, _ = oracle.count_cells(x, y, B, lins, tau - guard, band=0)
        b, _ = oracle.count_cells(x, y, B, lins, tau + guard, band=0)
        return a, b
    a, _ = oracle.count_cells(x, y, B, lins, tau, band=0)
    return a, None


def run_plan(x, y, eps, chain, levels, exchange=None, rank=0, world=1, excl=None, rho=0.0):
    """Run the planner to completion.  With world > 1 each rank counts its shard and
    `exchange(local_counts) -> list of per-rank arrays` gathers them (gloo).  excl / rho:
    exclusion balls (NEXT-2, rv_plan_create_ex)."""
    plan = rvmod.Plan(chain, levels, x.shape[0], eps, excl=excl, rho=rho)
    while True:
        req = plan.request()
        if req is None:
            break
        B, mode, lins = req
        if world == 1:
            a, b = oracle_counts(x, y, eps, B, mode, lins)
        else:
            lo, hi = rvmod.shard_range(lins.size, rank, world)
            la, lb = oracle_counts(x, y, eps, B, mode, lins[lo:hi])
            lb = lb if lb is not None else np.zeros_like(la)
            parts = exchange(np.stack([la, lb]) if la.size else np.zeros((2, 0), np.uint32))
            a = np.concatenate([p[0] for p in parts]).astype(np.uint32)
            b = np.concatenate([p[1] for p in parts]).astype(np.uint32)
            assert a.size == lins.size
        plan.feed(a, b)
    return plan.result()
