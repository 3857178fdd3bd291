"""cfg4-style problems over seeds (and cfg2/cfg3 variants): lb* from the dive vs the final
votes, per-phase block counts and time -- the certified search's robustness."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2506_11547_b200 import RotVote
which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
gen = getattr(datagen, which)
rv = RotVote(max_n=1_000_000)
for seed in range(int(sys.argv[2]) if len(sys.argv) > 2 else 8):
    pr = gen(seed=seed)
    x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
    rv.solve(x, y, pr.eps)
    r = rv.solve(x, y, pr.eps)
    print(which, "seed", seed, "ms %.2f" % r.ms, "votes", r.votes, "lb*", r.lb_star,
          "phases", r.cells_per_phase, flush=True)
