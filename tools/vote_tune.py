"""Tuning harness for the K3 vote kernel on the bench workload's levels (GPU only).

    python tools/vote_tune.py build          # (CPU) build variants into tools/bin/
    python tools/vote_tune.py run            # (GPU) time every variant x CTA shape
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {"base": {},
            "cpt8_v128_minb3": {"RV_CPT": 8, "RV_VOTERS": 128, "RV_MINB": 3},
            "cpt6_v128_minb4": {"RV_CPT": 6, "RV_VOTERS": 128, "RV_MINB": 4},
            "cpt4_v128_minb4": {"RV_CPT": 4, "RV_VOTERS": 128, "RV_MINB": 4},
            "cpt8_v128_minb3_s3": {"RV_CPT": 8, "RV_VOTERS": 128, "RV_MINB": 3, "RV_STAGES": 3},
            "cpt6_v192_minb2": {"RV_CPT": 6, "RV_VOTERS": 192, "RV_MINB": 2}}


def build():
    from paper_2506_11547_b200 import build as b
    os.makedirs(os.path.join(ROOT, "tools", "bin"), exist_ok=True)
    for tag, d in VARIANTS.items():
        b.build(out=os.path.join(ROOT, "tools", "bin", f"librotvote_{tag}.so"), defines=d)
        print("built", tag)


def one(tag, groups):
    """Runs in a subprocess with RV_LIB / RV_VOTE_GROUPS set."""
    import numpy as np
    import torch

    import datagen
    import oracle
    from paper_2506_11547_b200 import RV_MODE_BOUND, RotVote
    pr = datagen.cfg4()
    rv = RotVote(max_n=pr.n)
    x, y = torch.from_numpy(pr.x).cuda(), torch.from_numpy(pr.y).cuda()
    out = {"variant": tag, "groups": groups}
    for B in (45, 15, 90):
        lins = oracle.candidates(B)
        if B == 90:
            lins = lins[len(lins) // 2: len(lins) // 2 + 216]
        rv.count_cells(x, y, B, lins, pr.eps, RV_MODE_BOUND)   # warm
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            rv.count_cells(x, y, B, lins, pr.eps, RV_MODE_BOUND)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = min(ts)
        tf = len(lins) * pr.n * 18 / (ms * 1e-3) / 1e12
        out[f"B{B}_m{len(lins)}"] = {"ms": round(ms, 3), "tflops": round(tf, 2)}
    print(json.dumps(out), flush=True)


def run():
    for tag in VARIANTS:
        lib = os.path.join(ROOT, "tools", "bin", f"librotvote_{tag}.so")
        for g in (1, 4):
            env = dict(os.environ, RV_LIB=lib, RV_VOTE_GROUPS=str(g))
            subprocess.run([sys.executable, __file__, "one", tag, str(g)], env=env, timeout=300)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "build":
        build()
    elif cmd == "run":
        run()
    else:
        one(sys.argv[2], int(sys.argv[3]))
