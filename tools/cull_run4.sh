mkdir -p gpurun_out
timeout 300 python tools/cull_probe.py > gpurun_out/cull_probe.log 2>&1; echo "rc=$?" >> gpurun_out/cull_probe.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cull.csv python tools/trace_cfg4.py > gpurun_out/ncu_cull.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_cull.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rv_vote_cull_kernel -s 4 -c 1 -o gpurun_out/cull_l1 -f python tools/trace_cfg4.py > gpurun_out/ncu_cull_full.log 2>&1
