#!/bin/bash
# A/B of library variants in one GPU session: tools/ab_bench.sh "<bench args>" lib1 lib2 ...
# (an empty lib name = the in-tree librotvote.so).  Alternates the variants twice.
mkdir -p gpurun_out
ARGS="$1"; shift
for round in 1 2; do
  for lib in "$@"; do
    tag=$(basename "${lib:-current}" .so)
    RV_LIB=$lib timeout 300 python bench.py $ARGS --no-cpu-baseline > gpurun_out/ab_${tag}_$round.log 2>&1
    python - "$tag" "$round" <<'PY'
import json, sys
for l in open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.log"):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]
        print(f"{sys.argv[1]:24s} r{sys.argv[2]} ms/step {d['ms_per_step']:.3f} vote_ms {r['vote_ms_per_step']:.3f} "
              f"e2e_ms {d['e2e']['ms_per_step']:.2f} sm {d['clocks']['sm_mhz']}", flush=True)
PY
  done
done
