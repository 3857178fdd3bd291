"""Quick K3-TC check on the GPU: raw scores vs the oracle, counts vs the FFMA2 path, a solve."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen, oracle
from paper_2506_11547_b200 import RotVote, RV_MODE_BOUND, RV_MODE_BOUND_TC
oracle.build()
pr = datagen.make_problem(3000, 300, 0.01, 0.05, seed=1)
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=1 << 20, tensor_vote=True)
rng = np.random.default_rng(0)
for B in (15, 45, 360):
    lins = np.sort(rng.choice(oracle.candidates(B), 300, replace=False)).astype(np.uint32)
    sc = rv.debug_tc_scores(x, y, B, lins, pr.eps)
    errs = []
    for c in range(0, 300, 37):
        q = oracle.cell_quat(B, int(lins[c]))
        s = oracle.pair_stats(pr.x, pr.y, q)
        t = oracle.cell_bound_threshold(B, int(lins[c]), pr.eps) - 1e-5
        errs.append(np.abs(sc[c, :pr.n] - (s - t)).max())
        assert np.all(sc[c, pr.n:] == -1.0)
    print(f"B={B}: max |S'_tc - (s - t)| = {max(errs):.3e}", flush=True)
    a = rv.count_cells(x, y, B, lins, pr.eps, RV_MODE_BOUND_TC)
    b = rv.count_cells(x, y, B, lins, pr.eps, RV_MODE_BOUND)
    print(f"  counts tc vs ffma2: max diff {np.abs(a.astype(int) - b.astype(int)).max()}", flush=True)
ref = oracle.solve(pr.x, pr.y, pr.eps)
r = rv.solve(x, y, pr.eps)
print("solve tc", r.cell, r.votes, "oracle", ref.cell, ref.votes, r.cells_per_phase)
pr = datagen.cfg4()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv4 = RotVote(max_n=pr.n, tensor_vote=True)
rf = RotVote(max_n=pr.n)
for ctx, name in ((rv4, "tc"), (rf, "ffma2")):
    ctx.solve(x, y, pr.eps)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = ctx.solve(x, y, pr.eps)
    torch.cuda.synchronize()
    print(name, r.cell, r.votes, f"{1e3*(time.perf_counter()-t0):.2f} ms", f"vote {r.vote_ms:.2f} ms",
          r.cells_per_phase, flush=True)
