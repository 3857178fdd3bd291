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
VARIANTS = {"pipe0": {"RV_PIPE": 0}, "pipe0_s3": {"RV_PIPE": 0, "RV_STAGES": 3},
            "pipe0_asm": {"RV_PIPE": 0, "RV_COUNT_ASM": 1}, "pipe1": {"RV_PIPE": 1},
            "pipe1_asm": {"RV_PIPE": 1, "RV_COUNT_ASM": 1},
            "pipe0_cpt2_minb3": {"RV_PIPE": 0, "RV_CPT": 2, "RV_MINB": 3},
            "pipe0_t512_s2": {"RV_PIPE": 0, "RV_TILE": 512, "RV_STAGES": 2}}


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
