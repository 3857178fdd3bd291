"""Time cfg4 solves for several nested resolution chains (the certified result is chain-independent)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_2506_11547_b200 import RotVote
CHAINS = [(15, 45, 90, 180, 360), (15, 30, 90, 180, 360), (15, 30, 60, 120, 360), (10, 30, 90, 180, 360),
          (20, 60, 180, 360), (24, 72, 360), (30, 90, 180, 360), (12, 36, 72, 360), (15, 45, 180, 360),
          (15, 45, 90, 360), (20, 40, 120, 360), (18, 36, 72, 360), (15, 30, 90, 360)]
cfgs = sys.argv[1:] or ["cfg4"]
for cname in cfgs:
    pr = datagen.CONFIGS[cname]()
    x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
    ref = None
    for ch in CHAINS:
        for tc in (True,):
            rv = RotVote(max_n=pr.n, chain=ch, tensor_vote=tc)
            r = rv.solve(x, y, pr.eps, levels=len(ch))
            ts = []
            for _ in range(3):
                torch.cuda.synchronize(); t0 = time.perf_counter()
                r = rv.solve(x, y, pr.eps, levels=len(ch))
                ts.append(1e3 * (time.perf_counter() - t0))
            if ref is None: ref = (r.cell, r.votes)
            assert (r.cell, r.votes) == ref
            print(json.dumps({"cfg": cname, "chain": ch, "tc": tc, "ms": round(min(ts), 3),
                              "pair_votes": r.pair_votes, "cells": r.cells_per_phase}), flush=True)
            rv.close()
