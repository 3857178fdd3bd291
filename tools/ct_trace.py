"""Per-stage timeline of K3-CT in CTA 0 (tuning build with RV_CT_TRACE=1, loaded via RV_LIB):
runs the cfg4 level-1 culled vote and prints the per-stage intervals (clock64 cycles)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen, oracle
from paper_2506_11547_b200 import RotVote, rotvote
pr = datagen.cfg4()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n)
lins = oracle.candidates(45).astype(np.uint32)
for _ in range(2):
    rv.count_cells_culled(x, y, 15, 45, lins, pr.eps, 0)
torch.cuda.synchronize()
buf = np.zeros(7 * 4096, np.int64)
rotvote.lib().rv_ct_trace_copy(buf.ctypes.data_as(C.POINTER(C.c_longlong)), buf.size)
t = buf.reshape(7, 4096)
n = int((t[4] > 0).sum())
t0 = t[:, :n].min()
T = t[:, :n] - t0
names = ["gather start", "gather arrive", "mma full ok", "mma tempty ok", "mma commit",
         "epi tfull ok", "epi tempty arr"]
print("stages traced", n)
d = np.diff(T[4, 100:n - 1])
print("MMA commit period: median %d mean %.0f" % (np.median(d), d.mean()))
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6)]:
    v = T[b, 100:n - 100] - T[a, 100:n - 100]
    print(f"{names[a]:>15s} -> {names[b]:<15s}: median {np.median(v):8.0f}  p10 {np.percentile(v, 10):8.0f}  p90 {np.percentile(v, 90):8.0f}")
v = T[3, 102:n - 100] - T[6, 100:n - 102]
print("epi tempty arrive(k) -> mma tempty ok(k+2): median %.0f" % np.median(v))
print("first rows:")
for k in range(200, 212):
    print(k, [int(T[r, k]) for r in range(7)])
