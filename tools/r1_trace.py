"""Phase stamps (%globaltimer, CTA 0) of the fused refinement on cfg4; needs a library built
with -DRV_R1_TRACE=1 (RV_LIB=...)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_2506_11547_b200 import RotVote, rotvote
pr = datagen.cfg4()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n, chain=(15, 45, 180, 360))
for _ in range(4):
    r = rv.solve(x, y, pr.eps)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 32)()
rotvote.lib().rv_r1_trace_copy(buf)
t0 = buf[0]
names = ["q0", "q0 sync"] + [f"r{r} {w}" for r in range(3) for w in ("pass", "sync1", "eig", "sync2")]
for k in range(14):
    print(f"{names[k]:>10s} {(buf[k] - t0) / 1000:8.2f} us")
for r_ in range(3):
    print(f"  round {r_}: after sync1 -> loads {(buf[16+4*r_]-buf[3+4*r_])/1000:.2f} us, -> shuffles "
          f"{(buf[17+4*r_]-buf[16+4*r_])/1000:.2f}, -> syncthreads {(buf[18+4*r_]-buf[17+4*r_])/1000:.2f}, "
          f"-> eig done {(buf[4+4*r_]-buf[18+4*r_])/1000:.2f}")
print("refine phase ms", r.phase_ms["refine"])
