import sys, os
sys.path.insert(0, "/root/repo")
import torch, datagen
from paper_2506_11547_b200 import RotVote
bt = datagen.cfg5()
rv = RotVote(max_n=bt.x.shape[0], max_problems=4096)
x, y = torch.from_numpy(bt.x).cuda(), torch.from_numpy(bt.y).cuda()
for i in range(3):
    r = rv.solve_batched(x, y, bt.offsets, bt.eps)
    print("ms", r[0].ms, file=sys.stderr)
