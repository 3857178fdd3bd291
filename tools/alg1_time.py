"""Algorithm 1 (NEXT-4) on cfg4 vs the exact certified solve: times and rotation errors."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import datagen
from paper_2506_11547_b200 import RotVote
from scipy.spatial.transform import Rotation as Rot


def err(R, q):
    w, a, b, c = q
    return np.degrees((Rot.from_matrix(R).inv() * Rot.from_quat([a, b, c, w])).magnitude())


pr = datagen.cfg4()
rv = RotVote(max_n=pr.n)
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
for i in range(4):
    r = rv.alg1(x, y, J=180)
    s = rv.solve(x, y, pr.eps)
    print("alg1 ms %.3f (scatter %.3f) votes %d cell %s err %.4f deg | exact ms %.3f votes %d cell %s err %.4f deg"
          % (r["ms"], r["vote_ms"], r["votes"], r["cell"], err(pr.R, r["q"]), s.ms, s.votes, s.cell,
             err(pr.R, s.q)), flush=True)
