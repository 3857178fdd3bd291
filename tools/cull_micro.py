"""K3-C in isolation: the cfg4 level-1 workload (all 52,461 B=45 blocks against their B=15
ancestors' lists) through rot_vote_count_cells_culled; time = (all blocks) - (one block), CUDA
events.  RV_LIB selects a variant library.  Counts are checked against the base library's when
REF is set (a .npy path written by the base run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen, oracle
from paper_2506_11547_b200 import RotVote
pr = datagen.cfg4()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n)
lins = oracle.candidates(45).astype(np.uint32)
def t(l, reps=6):
    ts = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); c = rv.count_cells_culled(x, y, 15, 45, l, pr.eps, 0); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2], c
t1, _ = t(lins[:1])
ta, c = t(lins)
name = os.environ.get("NAME", "base")
print(f"{name}: all {ta:.3f} ms, one {t1:.3f} ms, K3-C ~ {ta - t1:.3f} ms, sum counts {int(c.sum())}")
