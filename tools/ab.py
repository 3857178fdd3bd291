"""A/B timing of compile-time variants of librotvote on the bench workload (cfg4, bench chain).
    python tools/ab.py build NAME=DEF:V,DEF:V ...   (here; side libraries in tools/bin/)
    python tools/ab.py run [--chain 15,45,180,360] NAME ...   (on the box; 'base' = in-tree lib)
Per variant: median over 15 solves (L2 flushed before each) of the solve's device time, the
culled-vote time (K3-CT) and the level-0 vote time (K3-TC), and the answer."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "bin")

CODE = r"""
import sys, torch, datagen, numpy as np
from paper_2506_11547_b200 import RotVote
chain = tuple(int(c) for c in sys.argv[1].split(","))
cfg = sys.argv[2]
pr = getattr(datagen, cfg)()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n, chain=chain, stream=torch.cuda.current_stream())
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ms, cm, vm, la, rs = [], [], [], [], []
for i in range(18):
    flush.zero_(); torch.cuda.synchronize()
    r = rv.solve(x, y, pr.eps)
    if i >= 3:
        ms.append(r.ms); cm.append(r.cull_ms); vm.append(r.vote_ms); la.append(r.launches); rs.append(r)
med = lambda v: sorted(v)[len(v) // 2]
l0 = med([v.phase_ms["level0"] for v in rs]) if rs and getattr(rs[0], "phase_ms", None) else 0.0
print(f"{sys.argv[3]:>10s} {cfg}: solve {med(ms):.3f} ms (min {min(ms):.3f})  level0 {l0:.3f}  K3-CT {med(cm):.3f}  "
      f"K3-TC {med(vm):.3f}  launches {la[-1]}  cell {r.cell} votes {r.votes} ties {r.n_tied}", flush=True)
"""


MICRO = r"""
import sys, torch, datagen, numpy as np, oracle
from paper_2506_11547_b200 import RotVote
pr = datagen.cfg4()
x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
rv = RotVote(max_n=pr.n)
lins = oracle.candidates(45).astype(np.uint32)
def t(l, reps=7):
    ts = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); c = rv.count_cells_culled(x, y, 15, 45, l, pr.eps, 0); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2], c
t1, _ = t(lins[:1])
ta, c = t(lins)
print(f"{sys.argv[1]:>10s} level-1 micro: all {ta:.3f} ms, one {t1:.3f} ms, culled vote ~ {ta - t1:.3f} ms, "
      f"sum counts {int(c.sum())}", flush=True)
"""


def build(specs):
    from paper_2506_11547_b200 import build as b
    os.makedirs(OUT, exist_ok=True)
    for spec in specs:
        name, _, defs = spec.partition("=")
        d = dict(kv.split(":") for kv in defs.split(",") if kv)
        b.build(out=os.path.join(OUT, f"librotvote_{name}.so"), defines=d)
        print("built", name, d)


def run(args):
    chain, cfg, micro = "15,45,180,360", "cfg4", False
    names = []
    it = iter(args)
    for a in it:
        if a == "--chain":
            chain = next(it)
        elif a == "--cfg":
            cfg = next(it)
        elif a == "--micro":
            micro = True
        else:
            names.append(a)
    for name in names:
        env = dict(os.environ)
        if name != "base":
            env["RV_LIB"] = os.path.join(OUT, f"librotvote_{name}.so")
        args = [MICRO, name] if micro else [CODE, chain, cfg, name]
        subprocess.run([sys.executable, "-c", *args], env=env, cwd=os.path.dirname(HERE),
                       timeout=int(os.environ.get("AB_TIMEOUT", "600")))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2:])
