"""Per-solve timing split of the culled path (cfg4 and a cfg5 batch): total, K3-TC, K3-C."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen
from paper_2506_11547_b200 import RotVote
pr = datagen.cfg4()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
for cull in (True, False):
    rv = RotVote(max_n=pr.n, cull=cull)
    for i in range(4):
        r = rv.solve(x, y, pr.eps)
    print(f"cfg4 cull={cull} ms={r.ms:.3f} tc_ms={r.vote_ms:.3f} cull_ms={r.cull_ms:.3f} "
          f"tc_pairs={r.vote_pairs:.3e} cull_pairs={r.cull_pairs:.3e} launches={r.launches} "
          f"cull_launches={r.cull_launches} phases={r.cells_per_phase}", flush=True)
    rv.close()
bt = datagen.cfg5(int(os.environ.get("P5", "4096")))
x, y = torch.from_numpy(bt.x).cuda(), torch.from_numpy(bt.y).cuda()
for cull in (True, False):
    rv = RotVote(max_n=int(bt.offsets[-1]), max_problems=len(bt.problems), cull=cull)
    for i in range(3):
        res = rv.solve_batched(x, y, bt.offsets, bt.eps, raw=True) if False else rv.solve_batched(x, y, bt.offsets, bt.eps)
    r = res[0]
    print(f"cfg5 cull={cull} ms={r.ms:.3f} tc_ms={r.vote_ms:.3f} cull_ms={r.cull_ms:.3f} "
          f"tc_pairs={r.vote_pairs:.3e} cull_pairs={r.cull_pairs:.3e} launches={r.launches}", flush=True)
    rv.close()
