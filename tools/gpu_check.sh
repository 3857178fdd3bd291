#!/bin/bash
# One GPU check pass: clocks/peaks microbench, smoke, GPU tests, bench.  Logs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 120 ./tools/bin/fma_peak > gpurun_out/fma_peak.txt 2>&1; echo "fma_peak rc=$?" >> gpurun_out/fma_peak.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
