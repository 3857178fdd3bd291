"""World-size-2 CPU tests (gloo) of the multi-rank path's host logic.

Single problem: every rank runs the library's planner; each request is sharded with the
library's rv_shard_range, each rank counts its own shard (exact counts from the CPU oracle
stand in for the GPU kernel), the shards are all-gathered over gloo exactly as
rot_vote_solve all-gathers them over NCCL, and both ranks must reach the world-1 result.
Batched: problems are range-sharded, solved independently and the results gathered."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        from paper_2506_11547_b200 import rotvote as rvmod
        from planner_util import run_plan

        def exchange(local):
            parts = [None] * world
            dist.all_gather_object(parts, local)
            return parts

        out = {}
        for name, pr, chain in (("cfg1", datagen.cfg1(), rvmod.DEFAULT_CHAIN),
                                ("small", datagen.make_problem(300, 30, 0.01, 0.08, seed=5),
                                 (5, 15, 45, 90))):
            r = run_plan(pr.x, pr.y, pr.eps, chain, 0, exchange=exchange, rank=rank, world=world)
            out[name] = (r.lin, r.votes, r.n_tied, r.pair_votes)
        # batched: contiguous problem ranges per rank, no per-level exchange
        probs = [datagen.make_problem(40 + 7 * p, 12, 0.02, 0.1, seed=[3, p]) for p in range(7)]
        lo, hi = rvmod.shard_range(len(probs), rank, world)
        mine = [run_plan(p.x, p.y, p.eps, (5, 15, 45), 0) for p in probs[lo:hi]]
        mine = [(r.lin, r.votes, r.n_tied) for r in mine]
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        out["batched"] = [t for part in parts for t in part]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_planner_matches_single_rank(world):
    import datagen
    import oracle
    from paper_2506_11547_b200 import build
    from paper_2506_11547_b200 import rotvote as rvmod
    from planner_util import run_plan
    build.build()
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # world-1 reference through the same planner, and the oracle's own search
    pr = datagen.cfg1()
    ref = oracle.solve(pr.x, pr.y, pr.eps)
    r1 = run_plan(pr.x, pr.y, pr.eps, rvmod.DEFAULT_CHAIN, 0)
    for rank in range(world):
        got = results[rank]
        assert got["cfg1"] == (r1.lin, r1.votes, r1.n_tied, r1.pair_votes)
        assert got["cfg1"][:3] == (ref.lin, ref.votes, ref.n_tied)
        assert got["small"] == results[0]["small"]
        assert got["batched"] == results[0]["batched"]
    probs = [datagen.make_problem(40 + 7 * p, 12, 0.02, 0.1, seed=[3, p]) for p in range(7)]
    want = []
    for p in probs:
        o = oracle.solve(p.x, p.y, p.eps, chain=(5, 15, 45), levels=3)
        want.append((o.lin, o.votes, o.n_tied))
    assert results[0]["batched"] == want
    _ = np
