"""Where does the one-pass refinement diverge from K6/K7?  Round by round on one problem."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import datagen
from paper_2506_11547_b200 import RotVote

pr = datagen.make_problem(4000, 400, 0.01, 0.05, seed=1)
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
for rounds in (0, 1, 2):
    a = RotVote(max_n=pr.n, refine_rounds=rounds)
    b = a.twin(planner="device_sync")
    ma = torch.zeros((pr.n + 31) // 32, dtype=torch.int32, device="cuda")
    mb = torch.zeros_like(ma)
    ra = a.solve(x, y, pr.eps, mask=ma)
    rb = b.solve(x, y, pr.eps, mask=mb)
    q, fl, ni = a.refine(x, y, pr.eps, rb.q_cell, rounds)
    print("rounds", rounds, "qcell eq", np.array_equal(ra.q_cell, rb.q_cell),
          "q eq", np.array_equal(ra.q, rb.q), "q-refine eq", np.array_equal(q, rb.q),
          "mask eq", torch.equal(ma, mb), "ninl", ra.n_inliers, rb.n_inliers, ni,
          "dq", np.abs(ra.q - rb.q).max(), "flags", ra.flags, rb.flags, fl, flush=True)
    a.close(); b.close()
