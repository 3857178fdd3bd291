"""cfg4 as a one-problem batch (the device level loop with P = 1): timings, RV_TRACE phases,
and with PROFILE_LAST=1 a profiler window around the last call."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import datagen
from paper_2506_11547_b200 import RotVote
pr = datagen.cfg4()
rv = RotVote(max_n=pr.n, tensor_vote=True)
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
offs = np.array([0, pr.n], np.int64)
prof = os.environ.get("PROFILE_LAST") == "1"
for i in range(4):
    if prof and i == 3:
        torch.cuda.profiler.start()
    r = rv.solve_batched(x, y, offs, pr.eps)[0]
    if prof and i == 3:
        torch.cuda.profiler.stop()
    s = rv.solve(x, y, pr.eps)
    print("batched-P1 ms %.3f vote %.3f launches %d | single ms %.3f vote %.3f launches %d | same %s"
          % (r.ms, r.vote_ms, r.launches, s.ms, s.vote_ms, s.launches,
             (r.cell, r.votes) == (s.cell, s.votes)), file=sys.stderr, flush=True)
