"""One small culled level in isolation (the 216 B=90 children of the best B=45 block of cfg4)
through rot_vote_count_cells_culled: the planner's one-CTA launch + the vote.  RV_LIB selects a
variant; run under ncu for per-kernel times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen, oracle
from paper_2506_11547_b200 import RotVote
pr = datagen.cfg4()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n)
i, j, k = 163 // 4, 101 // 4, 189 // 4   # the winner's B=90 block
lins = np.array([oracle.lin_of(90, i + a, j + b, k + c) for a in range(-3, 3) for b in range(-3, 3)
                 for c in range(-3, 3)], dtype=np.uint32)
for _ in range(5):
    c = rv.count_cells_culled(x, y, 15, 90, lins, pr.eps, 0)
print(os.environ.get("NAME", "base"), int(c.sum()))
