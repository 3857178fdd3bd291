"""Phase cycles of the one-CTA planner (cull_plan_small) over one cfg4 solve: a tuning build with
RV_PS_TIMING=1 (RV_LIB) prints them from the device."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_2506_11547_b200 import RotVote
pr = datagen.cfg4()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n, chain=(15, 45, 180, 360))
rv.solve(x, y, pr.eps)
torch.cuda.synchronize()
print("---- second solve (warm)", flush=True)
rv2 = RotVote(max_n=pr.n, chain=(15, 45, 180, 360))
rv2.solve(x, y, pr.eps)
torch.cuda.synchronize()
