"""A small one-pass solve under compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_2506_11547_b200 import RotVote
pr = datagen.make_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 2000, 200, 0.01, 0.05, seed=1)
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n, chain=(15, 45, 180, 360))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    r = rv.solve(x, y, pr.eps)
    print("cell", r.cell, "votes", r.votes, "syncs", r.host_syncs, flush=True)
