import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_2506_11547_b200 import RotVote
pr = datagen.cfg4()
rv = RotVote(max_n=pr.n, tensor_vote=True)
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
for i in range(3):
    r = rv.solve(x, y, pr.eps)
    print("ms", r.ms, "vote", r.vote_ms, file=sys.stderr, flush=True)
