"""Rigid pose over outlier ratios and seeds (paper's setting): time and errors per solve."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import datagen
from paper_2506_11547_b200 import RotVote
from scipy.spatial.transform import Rotation as Rot
rv = RotVote(max_n=4_000_000)
for rho in (0.9, 0.95, 0.97, 0.99):
    for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
        p = datagen.make_rigid(5000, rho, 0.01, seed=seed)
        x, y = torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda()
        rv.rigid(x, y, 0.05, 0.05)
        r = rv.rigid(x, y, 0.05, 0.05)
        w, a, b, c = r["q"]
        e = np.degrees((Rot.from_matrix(p.R).inv() * Rot.from_quat([a, b, c, w])).magnitude())
        print("rho %.2f seed %d ms %8.2f rot %.3f deg t %.4f kept %d" %
              (rho, seed, r["ms"], e, np.linalg.norm(r["t_mean"] - p.t), r["pairs_kept"]),
              flush=True)
