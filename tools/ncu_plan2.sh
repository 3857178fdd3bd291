mkdir -p gpurun_out
timeout 120 python tools/trace_cfg4.py > gpurun_out/plan_plain.log 2>&1 && \
timeout 600 ncu --set full --sampling-interval 0 --clock-control none --import-source on -k regex:cull_plan_small -s 10 -c 1 -o gpurun_out/prof_plan_small2 -f python tools/trace_cfg4.py > gpurun_out/ncu_plan.log 2>&1
echo rc=$? >> gpurun_out/ncu_plan.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cull_compact -s 2 -c 1 -o gpurun_out/prof_compact -f python tools/trace_cfg4.py > gpurun_out/ncu_compact.log 2>&1
echo rc=$? >> gpurun_out/ncu_compact.log
