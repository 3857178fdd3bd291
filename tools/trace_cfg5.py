import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_2506_11547_b200 import RotVote
tc = (sys.argv[1] if len(sys.argv) > 1 else "tc") == "tc"
bt = datagen.cfg5()
rv = RotVote(max_n=bt.x.shape[0], max_problems=4096, tensor_vote=tc)
x, y = torch.from_numpy(bt.x).cuda(), torch.from_numpy(bt.y).cuda()
for i in range(3):
    r = rv.solve_batched(x, y, bt.offsets, bt.eps)
    print("ms", r[0].ms, "vote_ms", r[0].vote_ms, file=sys.stderr, flush=True)
