"""Rigid pose (bench's scene) a few times on the library named by RV_LIB; prints after each call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_2506_11547_b200 import RotVote
rho = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
pr = datagen.make_rigid(5000, rho, 0.01, seed=0)
rv = RotVote(max_n=4_000_000, stream=torch.cuda.current_stream())
x = torch.from_numpy(pr.x).cuda()
y = torch.from_numpy(pr.y).cuda()
for i in range(5):
    r = rv.rigid(x, y, 0.05, 0.05)
    print(i, "ok ms %.3f rot_votes %d pairs %d" % (r["ms"], r["rot_votes"], r["pairs_kept"]), flush=True)
