"""The C-ABI library loads without a GPU and exports every function include/*.h declares;
the ctypes structs match the C layout."""
import ctypes as C
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2506_11547_b200 import build, rotvote
    build.build()
    return rotvote.lib()


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w \*]*?\b((?:rot_vote|rv)_\w+)\s*\(", src, re.M):
            names.add(m.group(1))
    return sorted(names)


def test_every_declared_symbol_is_exported(L):
    names = declared_functions()
    assert len(names) >= 15, names
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_struct_sizes_match_header(L):
    """Compile a tiny C program against include/rotvote.h and compare sizeof/offsetof."""
    import subprocess
    import tempfile
    from paper_2506_11547_b200 import rotvote as rv
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "rotvote.h"
#include "rotvote_plan.h"
int main(){printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(rv_config), sizeof(rv_result),
 sizeof(rv_plan_result), offsetof(rv_result, ms), offsetof(rv_config, stream),
 offsetof(rv_result, cells_per_phase), offsetof(rv_result, t_refine_ms));return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        got = [int(v) for v in subprocess.check_output([exe]).split()]
    want = [C.sizeof(rv.rv_config), C.sizeof(rv.rv_result), C.sizeof(rv.rv_plan_result),
            rv.rv_result.ms.offset, rv.rv_config.stream.offset, rv.rv_result.cells_per_phase.offset,
            rv.rv_result.t_refine_ms.offset]
    assert got == want


def test_create_without_gpu_fails_cleanly(L):
    """On a machine without a CUDA device, create reports an error instead of crashing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2506_11547_b200 import rotvote as rv
    cfg = rv.rot_vote_default_config()
    h = C.c_void_p()
    rc = L.rot_vote_create(C.byref(cfg), C.byref(h))
    assert rc in (rv.RV_ECUDA, rv.RV_ENOMEM) and not h.value
