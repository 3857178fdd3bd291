mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_cull.py tests/test_gpu_dplan.py -x -q -rf > gpurun_out/pytest_cull.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cull.log
( timeout 300 python tools/cull_ab.py run base
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_smem.csv python tools/trace_cfg4.py > /dev/null 2>&1; echo ncu rc=$? ) > gpurun_out/cull_ab15.log 2>&1
