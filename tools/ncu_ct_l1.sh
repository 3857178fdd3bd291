mkdir -p gpurun_out
PB="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $PB > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cull_tc \
    -s ${CT_SKIP:-21} -c 1 -o gpurun_out/prof_cull_tc -f $PB > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full.log
