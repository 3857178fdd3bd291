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
