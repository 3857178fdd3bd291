import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, datagen
from paper_2506_11547_b200 import RotVote, rotvote as rvm
from planner_util import run_plan
bt = datagen.cfg5(n_problems=8)
rv = RotVote(max_n=10000, max_problems=8)
x, y = torch.from_numpy(bt.x).cuda(), torch.from_numpy(bt.y).cuda()
res = rv.solve_batched(x, y, bt.offsets, bt.eps)
for p, r in zip(bt.problems, res):
    s = rv.solve(torch.from_numpy(p.x).cuda(), torch.from_numpy(p.y).cuda(), bt.eps)
    c = run_plan(p.x, p.y, bt.eps, rvm.DEFAULT_CHAIN, 0)
    print("batched", r.lb_star, r.cells_per_phase)
    print("single ", s.lb_star, s.cells_per_phase)
    print("cpu    ", c.lb_star, list(c.cells_per_phase[:c.n_phases]))
