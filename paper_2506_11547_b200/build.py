"""Build librotvote.so (sm_100a) in-tree with nvcc.

    python -m paper_2506_11547_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librotvote.so")
SOURCES = ["rv_kernels.cu", "rv_vote_tc.cu", "rv_dplan.cu", "rv_cull.cu", "rv_alg1.cu", "rv_rigid.cu",
           "rv_api.cpp", "rv_setup.cpp", "rv_host_plan.cpp", "rv_level_loop.cpp", "rv_plan.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    # every file of csrc/ and include/ (a header missing from a hand-kept list once left a stale
    # library in place)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps += [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: dict | None = None) -> str:
    """Build the library (out/defines: tuning variants, e.g. {"RV_CPT": 6})."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-Wall", "-I", os.path.join(ROOT, "include"),
           *[f"-D{k}={v}" for k, v in (defines or {}).items()],
           *[os.path.join(CSRC, f) for f in SOURCES], "-ldl", "-o", target + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
