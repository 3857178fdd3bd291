"""cfg3 two-peak solve with host-planner phase marks (RV_TRACE=1) and per-peak cell counts."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2506_11547_b200 import RotVote
pr = datagen.cfg3()
rv = RotVote(max_n=pr.n)
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
for i in range(2):
    res = rv.solve_multi(x, y, pr.eps, 2, 0.2)
    for r in res:
        print("peak", r.cell, r.votes, "cells_per_phase", r.cells_per_phase, "ms", r.ms,
              "vote_ms", r.vote_ms, file=sys.stderr, flush=True)
