"""Build K3-C variants (compile-time macros) as side libraries for A/B runs on the GPU box.
    python tools/cull_ab.py build NAME=DEFS ...   e.g. v1=RV_CULL_VARIANT:1 c3=RV_CULL_CTAS:3
    python tools/cull_ab.py run NAME ...          (on the box) -> cfg4 solve timing per variant"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "bin")


def build(specs):
    from paper_2506_11547_b200 import build as b
    os.makedirs(OUT, exist_ok=True)
    for spec in specs:
        name, _, defs = spec.partition("=")
        d = dict(kv.split(":") for kv in defs.split(",") if kv)
        b.build(out=os.path.join(OUT, f"librotvote_{name}.so"), defines=d)
        print("built", name, d)


def run(names):
    import subprocess
    for name in names:
        env = dict(os.environ)
        if name != "base":
            env["RV_LIB"] = os.path.join(OUT, f"librotvote_{name}.so")
        code = ("import torch, datagen\nfrom paper_2506_11547_b200 import RotVote\n"
                "pr = datagen.cfg4()\nx, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()\n"
                "rv = RotVote(max_n=pr.n)\nms=[]; cm=[]\n"
                "for i in range(12):\n    r = rv.solve(x, y, pr.eps)\n    ms.append(r.ms); cm.append(r.cull_ms)\n"
                "ms=sorted(ms[2:]); cm=sorted(cm[2:])\n"
                f"print('{name}', 'solve ms %.3f' % ms[len(ms)//2], 'cull ms %.3f' % cm[len(cm)//2], r.cell, r.votes)\n")
        subprocess.run([sys.executable, "-c", code], env=env, cwd=os.path.dirname(HERE))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        run(sys.argv[2:])
