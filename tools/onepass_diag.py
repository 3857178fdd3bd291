"""Per-kernel device times of one solve (torch.profiler / CUPTI) for the one-pass and the
per-level loop; phase times from rv_result.  Usage: python tools/onepass_diag.py [cfg4|n4000]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import datagen
from paper_2506_11547_b200 import RotVote

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
pr = datagen.cfg4() if which == "cfg4" else datagen.make_problem(4000, 400, 0.01, 0.05, seed=1)
chain = (15, 45, 180, 360) if which == "cfg4" else None
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
for planner in ("device", "device_sync"):
    rv = RotVote(max_n=pr.n, chain=chain, planner=planner)
    for _ in range(3):
        r = rv.solve(x, y, pr.eps)
    torch.cuda.synchronize()
    print(planner, "ms", round(r.ms, 3), "syncs", r.host_syncs, "launches", r.launches,
          "phases", {k: round(v, 3) for k, v in (r.phase_ms or {}).items()},
          "cells", r.cells_per_phase, "flags", r.flags, flush=True)
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        r = rv.solve(x, y, pr.eps)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    tot = 0.0
    for e in evs:
        d = e.device_time if hasattr(e, "device_time") else e.cuda_time
        tot += d
        print(f"   {d:9.1f} us  {e.name[:90]}")
    print(planner, "kernel sum us", round(tot, 1), "n", len(evs), flush=True)
    rv.close()
