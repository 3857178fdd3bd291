"""The 99%-outlier rigid case: per-phase block counts and times of the rotation vote."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import datagen
import oracle
from paper_2506_11547_b200 import RotVote
pr = datagen.make_rigid(5000, 0.99, 0.01, seed=0)
ij, m, d = oracle.rigid_pairs(pr.x, pr.y, 0.05)
rv = RotVote(max_n=4_000_000)
mm, dd = torch.from_numpy(m).cuda(), torch.from_numpy(d).cuda()
for i in range(2):
    r = rv.solve(mm, dd, 0.05)
    print("ms", r.ms, "vote_ms", r.vote_ms, "votes", r.votes, "lb*", r.lb_star, "rechecked",
          r.n_rechecked, "phases", r.cells_per_phase, "pairs", r.vote_pairs, file=sys.stderr,
          flush=True)
