"""cfg4 over seeds: the default solve (K3-CT culled levels), the FP32 culled solve (K3-C,
cull="fp32") and the unculled tensor-core solve must agree on (cell, votes, ties, q); prints
the three solve times.  Usage: python tools/cull_seed_check.py [cfg4] [n_seeds]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import datagen
from paper_2506_11547_b200 import RotVote

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
nseeds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
gen = getattr(datagen, which)
ct = RotVote(max_n=1_000_000)
k3c = RotVote(max_n=1_000_000, cull="fp32")
dense = RotVote(max_n=1_000_000, cull=False)
bad = 0
for seed in range(nseeds):
    pr = gen(seed=seed)
    x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
    rs = []
    for rv in (ct, k3c, dense):
        rv.solve(x, y, pr.eps)
        rv.solve(x, y, pr.eps)  # (captured)
        rs.append(rv.solve(x, y, pr.eps))  # (replayed)
    same = all((r.cell, r.votes, r.n_tied) == (rs[2].cell, rs[2].votes, rs[2].n_tied)
               and np.allclose(r.q, rs[2].q, atol=1e-12) for r in rs[:2])
    bad += not same
    print(which, "seed", seed, "K3-CT %.2f ms" % rs[0].ms, "K3-C %.2f ms" % rs[1].ms,
          "dense %.2f ms" % rs[2].ms, "votes", rs[0].votes, "retried" if rs[0].flags & 8 else "one pass",
          "same" if same else "DIFFERENT",
          flush=True)
print("mismatches", bad)
sys.exit(1 if bad else 0)
