mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cull.py -x -q -rf > gpurun_out/pytest_cull.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cull.log
timeout 300 python tools/cull_probe.py > gpurun_out/cull_probe.log 2>&1; echo "rc=$?" >> gpurun_out/cull_probe.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cull.csv python tools/trace_cfg4.py > gpurun_out/ncu_cull.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_cull.log
