"""Batched config 5 (4096 x 1000): three solves with their timings (RV_TRACE=1 adds the host
phase marks).  PROFILE_LAST=1 brackets the last solve with cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2506_11547_b200 import RotVote
tc = (sys.argv[1] if len(sys.argv) > 1 else "tc") == "tc"
bt = datagen.cfg5()
rv = RotVote(max_n=bt.x.shape[0], max_problems=4096, tensor_vote=tc)
x, y = torch.from_numpy(bt.x).cuda(), torch.from_numpy(bt.y).cuda()
prof = os.environ.get("PROFILE_LAST") == "1"
for i in range(3):
    if prof and i == 2:
        torch.cuda.profiler.start()
    r = rv.solve_batched(x, y, bt.offsets, bt.eps)
    if prof and i == 2:
        torch.cuda.profiler.stop()
    print("ms", r[0].ms, "vote_ms", r[0].vote_ms, "launches", r[0].launches, file=sys.stderr,
          flush=True)
