"""cfg4 over seeds with two chains: identical answers, per-chain solve time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen
from paper_2506_11547_b200 import RotVote
chains = [tuple(int(v) for v in c.split("-")) for c in (sys.argv[2] if len(sys.argv) > 2 else "15-45-90-180-360,15-45-180-360").split(",")]
rvs = [RotVote(max_n=1_000_000, chain=c) for c in chains]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
tot = [0.0] * len(chains); bad = 0
for seed in range(n):
    pr = datagen.cfg4(seed=seed)
    x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
    rs = []
    for rv, c in zip(rvs, chains):
        rv.solve(x, y, pr.eps, levels=len(c))
        ms = min(rv.solve(x, y, pr.eps, levels=len(c)).ms for _ in range(3))
        rs.append((rv.solve(x, y, pr.eps, levels=len(c)), ms))
    same = all((r[0].cell, r[0].votes) == (rs[0][0].cell, rs[0][0].votes) for r in rs)
    bad += not same
    for q, r in enumerate(rs): tot[q] += r[1]
    print(seed, " ".join(["%.3f"] * len(rs)) % tuple(r[1] for r in rs), "same" if same else "DIFFERENT", flush=True)
print("chains", chains, "mean ms", [t / n for t in tot], "mismatches", bad)
