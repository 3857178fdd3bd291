"""Small solves of every path, for compute-sanitizer (one tool per run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen
from paper_2506_11547_b200 import RotVote, RV_MODE_BOUND, RV_MODE_FINAL, RV_MODE_EXACT
pr = datagen.make_problem(3000, 300, 0.01, 0.05, seed=2)
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
for tc in (True, False):
    rv = RotVote(max_n=1 << 14, max_problems=16, tensor_vote=tc)
    mask = torch.zeros((pr.n + 31) // 32, dtype=torch.int32, device="cuda")
    r = rv.solve(x, y, pr.eps, mask=mask)
    print("solve", tc, r.cell, r.votes, flush=True)
    probs = [datagen.make_problem(300 + 50 * p, 40, 0.02, 0.09, seed=[1, p]) for p in range(5)]
    bt = datagen.batch_of(probs, 0.09)
    rs = rv.solve_batched(torch.from_numpy(bt.x).cuda(), torch.from_numpy(bt.y).cuda(), bt.offsets, bt.eps)
    print("batched", tc, [q.votes for q in rs], flush=True)
    lins = np.arange(0, 2295, 7, dtype=np.uint32)
    for mode in (RV_MODE_BOUND, RV_MODE_FINAL, RV_MODE_EXACT):
        rv.count_cells(x, y, 15, lins, pr.eps, mode)
    rv.close()
print("done")
