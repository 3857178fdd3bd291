#!/bin/bash
# ncu full captures of two vote launches of one solve (level 0 and the large level-1 launch),
# each after a clean plain run of the same command.  Output: gpurun_out/prof_vote_{l0,big}.ncu-rep
mkdir -p gpurun_out
PB="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $PB > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rv_vote_kernel \
    -s 0 -c 1 -o gpurun_out/prof_vote_l0 -f $PB > gpurun_out/ncu_l0.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_l0.log
timeout 300 $PB > gpurun_out/ncu_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rv_vote_kernel \
    -s 5 -c 1 -o gpurun_out/prof_vote_big -f $PB > gpurun_out/ncu_big.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_big.log
timeout 300 $PB > gpurun_out/ncu_plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $PB > gpurun_out/ncu_launches.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launches.log
