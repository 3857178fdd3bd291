mkdir -p gpurun_out
timeout 120 python tools/trace_cfg4.py > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rv_vote_cull_kernel -s 4 -c 1 -o gpurun_out/cull_l1 -f python tools/trace_cfg4.py > gpurun_out/ncu_cull_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_cull_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cull_compact -c 1 -o gpurun_out/cull_compact -f python tools/trace_cfg4.py > gpurun_out/ncu_compact_full.log 2>&1
