"""Time the K3-TC big level under stage ablations (RV_TC_ABLATE bits: 1 count, 2 MMA, 4 TMA)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1:
    import numpy as np, torch, datagen, oracle
    from paper_2506_11547_b200 import RotVote, RV_MODE_BOUND_TC
    pr = datagen.cfg4()
    x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
    rv = RotVote(max_n=pr.n, tensor_vote=True)
    lins = oracle.candidates(45)
    rv.count_cells(x, y, 45, lins, pr.eps, RV_MODE_BOUND_TC)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); rv.count_cells(x, y, 45, lins, pr.eps, RV_MODE_BOUND_TC); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"ablate": int(sys.argv[1]), "ms": min(ts)}), flush=True)
else:
    for a in [int(v) for v in os.environ.get("ABL_LIST", "0,1,2,4,3,6,5,7").split(",")]:
        subprocess.run([sys.executable, __file__, str(a)], env=dict(os.environ, RV_TC_ABLATE=str(a)), timeout=300)
