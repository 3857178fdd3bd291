"""Per-kernel device time of one batched cfg5 solve (torch.profiler / CUPTI), grouped by name."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2506_11547_b200 import RotVote

bt = datagen.cfg5()
x, y = torch.from_numpy(bt.x).cuda(), torch.from_numpy(bt.y).cuda()
cull = sys.argv[1] if len(sys.argv) > 1 else "on"
rv = RotVote(max_n=bt.x.shape[0], max_problems=4096, cull=(cull == "on"))
for _ in range(3):
    res = rv.solve_batched(x, y, bt.offsets, bt.eps)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    res = rv.solve_batched(x, y, bt.offsets, bt.eps)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0])
tot = 0.0
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    d = e.device_time
    tot += d
    k = e.name.split("(")[0][:70]
    agg[k][0] += d
    agg[k][1] += 1
for k, (d, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{d:9.1f} us {c:4d}x  {k}")
print("kernel sum us", round(tot, 1), "solve ms", res[0].ms, "votes[0]", res[0].votes)
