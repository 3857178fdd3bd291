"""CPU tests of librotvote's host logic: the certified-search planner (driven by exact
oracle counts), the shard ranges and the candidate grid.  No GPU needed: these entry
points are plain C++ (include/rotvote_plan.h)."""
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


@pytest.mark.parametrize("B", [1, 3, 5, 15, 45, 90])
def test_grid_candidates_match_oracle(B):
    assert np.array_equal(rvmod.grid_candidates(B), oracle.candidates(B))


def test_shard_range_partitions():
    for m in (0, 1, 7, 2295, 52461):
        for W in (1, 2, 3, 4, 8):
            spans = [rvmod.shard_range(m, r, W) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


CHAINS = [(3, 9, 27), (5, 15, 45), (4, 8, 16, 32), (2, 4, 8, 16), (6, 18)]


def test_planner_equals_exhaustive_random():
    rng = np.random.default_rng(21)
    for trial in range(120):
        n = int(rng.integers(2, 50))
        eps = float(rng.choice([0.03, 0.1, 0.4, 1.2, 2.8]))
        pr = datagen.make_problem(n, int(rng.integers(0, n + 1)), float(rng.choice([0, .01, .05])),
                                  eps, seed=int(rng.integers(1 << 30)))
        x, y = pr.x, pr.y
        if trial % 5 == 1:
            y[: n // 2] = -x[: n // 2]
        chain = CHAINS[trial % len(CHAINS)]
        ex = oracle.solve(x, y, eps, chain=chain, levels=len(chain), exhaustive=True)
        for L in range(1, len(chain) + 1):
            r = run_plan(x, y, eps, chain, L)
            assert (r.lin, r.votes, r.n_tied) == (ex.lin, ex.votes, ex.n_tied), (trial, chain, L)
            assert r.B == chain[-1]


def test_planner_cfg1_default_chain():
    pr = datagen.cfg1()
    ref = oracle.solve(pr.x, pr.y, pr.eps)      # certified == exhaustive (pinned elsewhere)
    for L in (0, 2, 5, 6):
        r = run_plan(pr.x, pr.y, pr.eps, rvmod.DEFAULT_CHAIN, L)
        assert (r.lin, r.votes, r.n_tied) == (ref.lin, ref.votes, ref.n_tied)
        assert r.lb_star <= r.votes


def test_planner_rejects_bad_arguments():
    with pytest.raises(ValueError):
        rvmod.Plan((5, 16), 2, 10, 0.1)         # 16 not divisible by 5
    with pytest.raises(ValueError):
        rvmod.Plan((5, 15), 3, 10, 0.1)         # levels > chain length
    with pytest.raises(ValueError):
        rvmod.Plan((5, 15), 2, 10, 0.0)         # eps not in (0, pi)
    with pytest.raises(ValueError):
        rvmod.Plan((5, 15), 2, 10, 3.2)


def test_planner_request_protocol():
    pr = datagen.make_problem(30, 10, 0.01, 0.1, seed=3)
    plan = rvmod.Plan((5, 15, 45), 3, 30, 0.1)
    B, mode, lins = plan.request()
    assert B == 5 and mode == rvmod.RV_MODE_BOUND and np.all(np.diff(lins.astype(np.int64)) > 0)
    with pytest.raises(ValueError):
        plan.result()


def test_planner_external_level0_protocol():
    """rv_plan_feed_l0_start / rv_plan_feed_l0_survivors (the batched solve's device-side
    level-0 reduction) reach the same result and cells as feeding level 0 directly."""
    import ctypes as C
    from planner_util import oracle_counts
    L = rvmod.lib()
    L.rv_plan_feed_l0_start.argtypes = [C.c_void_p, C.c_int64]
    L.rv_plan_needs_l0_survivors.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    L.rv_plan_feed_l0_survivors.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    L.rv_plan_l0_background.argtypes = [C.c_int32, C.c_double, C.POINTER(C.c_int64)]
    L.rv_plan_l0_background.restype = C.POINTER(C.c_double)
    rng = np.random.default_rng(31)
    for trial in range(25):
        n = int(rng.integers(5, 400))
        eps = float(rng.choice([0.05, 0.1, 0.3]))
        pr = datagen.make_problem(n, n // 4, 0.01, eps, seed=int(rng.integers(1 << 30)))
        chain = (5, 15, 45, 90)
        ref = run_plan(pr.x, pr.y, eps, chain, 0)
        plan = rvmod.Plan(chain, 0, n, eps)
        B, mode, lins = plan.request()
        ub, _ = oracle_counts(pr.x, pr.y, eps, B, mode, lins)
        m = C.c_int64()
        bgp = L.rv_plan_l0_background(B, eps, C.byref(m))
        bg = np.ctypeslib.as_array(bgp, shape=(m.value,))
        # the documented key: centre inside first, then max excess, ties -> lowest index
        ijk = np.stack([lins // (B * B), (lins // B) % B, lins % B], 1).astype(np.int64)
        inside = (((2 * ijk + 1 - B) ** 2).sum(1) <= B * B)
        excess = ub.astype(np.float64) - float(n) * bg
        order = sorted(range(lins.size), key=lambda e: (-int(inside[e]), -excess[e], e))
        assert L.rv_plan_feed_l0_start(plan.h, order[0]) == 0
        while True:
            lb = C.c_int64()
            if L.rv_plan_needs_l0_survivors(plan.h, C.byref(lb)):
                surv = np.flatnonzero(ub.astype(np.int64) >= lb.value).astype(np.int32)
                assert L.rv_plan_feed_l0_survivors(plan.h, surv.ctypes.data, surv.size) == 0
                continue
            req = plan.request()
            if req is None:
                break
            B2, mode2, l2 = req
            a, b = oracle_counts(pr.x, pr.y, eps, B2, mode2, l2)
            plan.feed(a, b)
        r = plan.result()
        assert (r.lin, r.votes, r.n_tied, r.cells_evaluated) == (ref.lin, ref.votes, ref.n_tied,
                                                                 ref.cells_evaluated)
