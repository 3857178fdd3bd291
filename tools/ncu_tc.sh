#!/bin/bash
# ncu of the K3-TC launches of one solve (after a clean plain run): full capture of the big
# level-1 launch + the launch list.
mkdir -p gpurun_out
PB="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $PB > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rv_vote_tc \
    -s 5 -c 1 -o gpurun_out/prof_tc_big -f $PB > gpurun_out/ncu_tc_big.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_tc_big.log
timeout 300 $PB > gpurun_out/ncu_plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_tc.csv $PB > gpurun_out/ncu_launches.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launches.log
