mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cull.py -q -x > gpurun_out/pt.log 2>&1
timeout 300 python tools/cull_probe.py > gpurun_out/cull_probe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cull_compact -c 1 -o gpurun_out/cull_compact -f python tools/trace_cfg4.py > gpurun_out/ncu_compact_full.log 2>&1
