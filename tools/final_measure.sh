# Round-end measurement pass (one GPU): smoke, bench (default: cfg4 + cpu_baseline), the ncu
# launch list of a short bench run, ncu --set full of K3-CT's level-1 launch and of K3-TC's
# level-0 launch, cfg5 and NEXT-2 lines.  Everything lands in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
PB="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $PB > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $PB > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cull_tc \
    -s ${CT_SKIP:-21} -c 1 -o gpurun_out/prof_cull_tc_l1 -f $PB > gpurun_out/ncu_full_ct.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_ct.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rv_vote_tc_kernel \
    -s 3 -c 1 -o gpurun_out/prof_tc_l0 -f $PB > gpurun_out/ncu_full_tc.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_full_tc.log
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
timeout 300 python bench.py --method multi --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_multi.log 2>&1
