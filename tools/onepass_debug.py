"""Run one-pass solves of a config (debug builds via RV_LIB), printing every result."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_2506_11547_b200 import RotVote
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
chain = tuple(int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "15,45,180,360").split(","))
pr = getattr(datagen, cfg)()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n, chain=chain)
for i in range(4):
    r = rv.solve(x, y, pr.eps)
    print(i, "cell", r.cell, "votes", r.votes, "syncs", r.host_syncs, "flags", r.flags,
          "phases", r.cells_per_phase, flush=True)
