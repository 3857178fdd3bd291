#!/bin/bash
# One GPU check pass.  Logs -> gpurun_out/.  Env: PYTEST_MARK (default "gpu"), BENCH_ARGS,
# NCU=1 (launch list + full capture of the largest vote launch after a clean plain run).
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
BARGS=${BENCH_ARGS:---steps 10 --warmup 3}
if [ "${NCU:-0}" = "1" ]; then
  PB="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
  timeout 300 $PB > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $PB > gpurun_out/ncu_launches.log 2>&1
  echo "ncu launches rc=$?" >> gpurun_out/ncu_launches.log
  timeout 300 $PB > gpurun_out/ncu_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rv_vote_kernel \
      -s ${NCU_SKIP:-5} -c 1 -o gpurun_out/prof_vote -f $PB > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m "${PYTEST_MARK:-gpu}" -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py $BARGS > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
