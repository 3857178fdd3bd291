"""World-size-2/3 CPU tests (gloo) of the DEFAULT multi-rank path's partition logic: one
culled problem split over ranks (rotvote_plan.h rv_cull_partition).

Every rank takes the library's level-0 slice (whole ancestor groups per slice) and group
ownership; exact counts from the CPU oracle stand in for the GPU kernels:
  level 0   rank r counts the bound test of its slice's rows; one all_reduce(sum) over gloo
            assembles the level (vote_level0_slabs does the same with ncclAllReduce);
  lists     rank r builds the union lists of the groups it owns -- only from its
            own level-0 rows, so every member of an owned group must lie in its slice;
  level 1   rank r counts every finer block whose ancestor group it owns over that group's
            union list; one all_reduce(sum) (vote_level_owned).
The assembled counts must equal the one-rank culled counts, each block must be counted by
exactly one rank, and the culled counts must contain every true voter of the block (far pairs
decided as the oracle's unculled count)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B0, B1, SHAPE = 5, 15, (1, 2, 2)
GUARD = 1e-5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def culled_counts(pr, owned_groups, rows_mine):
    """Level-0 bound counts of rows_mine and the level-1 culled bound counts of the blocks whose
    ancestor group is in owned_groups (the rest zero).  Oracle arithmetic only."""
    import oracle
    from paper_2506_11547_b200 import rotvote as rvmod
    g_of, goff, gmem = rvmod.cull_groups(B0, SHAPE)
    l0 = oracle.candidates(B0)
    thr0 = np.array([oracle.cell_bound_threshold(B0, int(l), pr.eps) for l in l0]) - GUARD
    c0 = np.zeros(l0.size, np.int64)
    lists = {}
    for a in rows_mine:
        cnt, _ = oracle.count_cells(pr.x, pr.y, B0, l0[a:a + 1], thr0[a], band=0)
        c0[a] = int(cnt[0])
    # the pass list of a level-0 row: correspondences whose exact score clears its bound test
    xn = pr.x.astype(np.float64)
    yn = pr.y.astype(np.float64)
    xn /= np.linalg.norm(xn, axis=1, keepdims=True)
    yn /= np.linalg.norm(yn, axis=1, keepdims=True)
    for g in owned_groups:
        members = gmem[goff[g]:goff[g + 1]]
        assert all(a in rows_mine for a in members), "a group straddles two slices"
        U = np.zeros(pr.n, bool)
        for a in members:
            s = oracle.pair_stats(pr.x, pr.y, oracle.cell_quat(B0, int(l0[a])))
            U |= s >= thr0[a]
        lists[g] = np.flatnonzero(U)
    l1 = oracle.candidates(B1)
    f = B1 // B0
    row_of = {int(l): a for a, l in enumerate(l0)}
    c1 = np.zeros(l1.size, np.int64)
    own1 = np.zeros(l1.size, np.int64)
    for b, lin in enumerate(l1):
        i, j, k = lin // (B1 * B1), (lin // B1) % B1, lin % B1
        anc = row_of[int(((i // f) * B0 + j // f) * B0 + k // f)]
        g = int(g_of[anc])
        if g not in lists:
            continue
        U = lists[g]
        own1[b] = 1
        if U.size:
            t = oracle.cell_bound_threshold(B1, int(lin), pr.eps) - GUARD
            cnt, _ = oracle.count_cells(pr.x[U], pr.y[U], B1, [lin], t, band=0)
            c1[b] = int(cnt[0])
    return c0, c1, own1


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        from paper_2506_11547_b200 import rotvote as rvmod
        pr = datagen.make_problem(400, 60, 0.01, 0.08, seed=31)
        sl, gsl = rvmod.cull_partition(B0, world, SHAPE)
        rows = set(range(int(sl[rank]), int(sl[rank + 1])))
        owned = list(range(int(gsl[rank]), int(gsl[rank + 1])))
        c0, c1, own1 = culled_counts(pr, owned, rows)
        t0, t1, to = (torch.from_numpy(v) for v in (c0, c1, own1))
        for t in (t0, t1, to):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        q.put((rank, (sl.tolist(), gsl.tolist(), t0.numpy(), t1.numpy(), to.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split_problem_partition(world):
    import datagen
    import oracle
    from paper_2506_11547_b200 import build
    from paper_2506_11547_b200 import rotvote as rvmod
    build.build()
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sl, gsl = res[0][0], res[0][1]
    m0 = oracle.candidates(B0).size
    G = rvmod.cull_groups(B0, SHAPE)[1].size - 1
    assert sl[0] == 0 and sl[-1] == m0 and gsl[0] == 0 and gsl[-1] == G
    assert all(a <= b for a, b in zip(sl, sl[1:])) and all(a <= b for a, b in zip(gsl, gsl[1:]))
    assert max(b - a for a, b in zip(sl, sl[1:])) <= math.ceil(m0 / world) + 2 * B0  # balance
    # one-rank reference: every row, every group
    pr = datagen.make_problem(400, 60, 0.01, 0.08, seed=31)
    c0, c1, own1 = culled_counts(pr, range(G), set(range(m0)))
    for r in range(world):
        _, _, t0, t1, to = res[r]
        assert np.array_equal(t0, c0) and np.array_equal(t1, c1)
        assert np.all(to == 1)  # every finer block voted by exactly one rank
    # culled counts contain every true voter: >= the oracle's unculled count at t + guard
    l1 = oracle.candidates(B1)
    t = np.array([oracle.cell_bound_threshold(B1, int(l), pr.eps) for l in l1])
    far, _ = oracle.count_cells(pr.x, pr.y, B1, l1, t + GUARD, band=0)
    full, _ = oracle.count_cells(pr.x, pr.y, B1, l1, t - GUARD, band=0)
    assert np.all(c1 >= far) and np.all(c1 <= full)
    assert c1.max() >= 60 * 0.9  # the inlier block is found


# ---- the one-pass split solve: each rank searches the subtrees of its own groups ------------
CHAIN = (5, 15, 45)


def _children(B, lin, f):
    import oracle
    i, j, k = lin // (B * B), (lin // B) % B, lin % B
    Bc = B * f
    return [oracle.lin_of(Bc, f * i + a, f * j + b, f * k + c)
            for a in range(f) for b in range(f) for c in range(f)
            if oracle.cell_is_candidate(Bc, f * i + a, f * j + b, f * k + c)]


def subtree_search(pr, owned_groups, lb):
    """The branch and bound over the subtrees of owned_groups' level-0 blocks (bounds: the
    oracle's exact UB counts at cos(eps + r(c)) - guard; finest level: exact counts), from the
    certified lower bound lb.  Returns the local winner key (count << 32 | ~lin), its ties, and
    the finest blocks it decided.  Oracle arithmetic only."""
    import oracle
    from paper_2506_11547_b200 import rotvote as rvmod
    g_of = rvmod.cull_groups(CHAIN[0], SHAPE)[0]
    l0 = oracle.candidates(CHAIN[0])
    level = [int(l) for a, l in enumerate(l0) if int(g_of[a]) in owned_groups]
    for li in range(len(CHAIN) - 1):
        B = CHAIN[li]
        thr = np.array([oracle.cell_bound_threshold(B, l, pr.eps) for l in level]) - GUARD
        ub, _ = oracle.count_cells(pr.x, pr.y, B, level, thr, band=0) if level else ([], None)
        level = [l for l, u in zip(level, ub) if u >= lb]
        f = CHAIN[li + 1] // B
        level = [c for l in level for c in _children(B, l, f)]
    Bf = CHAIN[-1]
    if not level:
        return 0, 0, set()
    cnt, _ = oracle.count_cells(pr.x, pr.y, Bf, level, math.cos(pr.eps), band=0)
    best = max((int(c) << 32) | (0xFFFFFFFF - int(l)) for c, l in zip(cnt, level))
    ties = int(np.sum(cnt == (best >> 32)))
    return best, ties, set(level)


def _worker_subtree(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import oracle
        from paper_2506_11547_b200 import rotvote as rvmod
        pr = datagen.make_problem(300, 60, 0.01, 0.08, seed=41)
        _, gsl = rvmod.cull_partition(CHAIN[0], world, SHAPE)
        owned = set(range(int(gsl[rank]), int(gsl[rank + 1])))
        # a certified lower bound every rank computes alike (the replicated dive's role): the
        # exact count of the finest block that holds the ground-truth rotation
        p = oracle.project(oracle.canonicalize(_quat_of_R(pr.R)))
        B = CHAIN[-1]
        ijk = [min(B - 1, max(0, int((v + 1.0) * B / 2.0))) for v in p]
        lb = int(oracle.count_cells(pr.x, pr.y, B, [oracle.lin_of(B, *ijk)],
                                    math.cos(pr.eps), band=0)[0][0])
        best, ties, mine = subtree_search(pr, owned, lb)
        # the merge: every rank's (key, ties), the largest key, the ties of equal counts
        keys = [None] * world
        dist.all_gather_object(keys, (best, ties, sorted(mine)))
        gbest = max(k[0] for k in keys)
        gties = sum(k[1] for k in keys if k[0] and (k[0] >> 32) == (gbest >> 32))
        q.put((rank, (gbest, gties, [k[2] for k in keys], lb)))
    finally:
        dist.destroy_process_group()


def _quat_of_R(R):
    """Scalar-first unit quaternion of a rotation matrix (test helper, Shepperd's method)."""
    t = np.trace(R)
    if t > 0:
        s = 2.0 * math.sqrt(1.0 + t)
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
    else:
        i = int(np.argmax(np.diag(R)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = 2.0 * math.sqrt(1.0 + R[i, i] - R[j, j] - R[k, k])
        q = [0.0] * 4
        q[0] = (R[k, j] - R[j, k]) / s
        q[1 + i] = 0.25 * s
        q[1 + j] = (R[j, i] + R[i, j]) / s
        q[1 + k] = (R[k, i] + R[i, k]) / s
    q = np.array(q)
    return q / np.linalg.norm(q)


@pytest.mark.parametrize("world", [2, 3])
def test_split_problem_subtree_search(world):
    """The one-pass split solve's branch and bound: rank r searches only the subtrees of the
    level-0 groups it owns, from a lower bound every rank shares, with no collective; merging
    the ranks' (winner key, ties) gives the one-rank certified result (= the oracle's exhaustive
    optimum), and every decided finest block belongs to exactly one rank."""
    import datagen
    import oracle
    from paper_2506_11547_b200 import build
    build.build()
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_subtree, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pr = datagen.make_problem(300, 60, 0.01, 0.08, seed=41)
    ref = oracle.solve(pr.x, pr.y, pr.eps, chain=CHAIN)
    one_best, one_ties, one_set = subtree_search(pr, set(range(10 ** 6)), res[0][3])
    for r in range(world):
        gbest, gties, sets, lb = res[r]
        assert lb >= 1 and lb <= ref.votes  # a certified lower bound that prunes
        votes, lin = gbest >> 32, 0xFFFFFFFF - (gbest & 0xFFFFFFFF)
        assert (votes, lin, gties) == (ref.votes, ref.lin, ref.n_tied)
        assert (gbest, gties) == (one_best, one_ties)
        union = set().union(*map(set, sets))
        assert sum(len(s) for s in sets) == len(union) == len(one_set)  # disjoint, complete
        assert union == one_set
