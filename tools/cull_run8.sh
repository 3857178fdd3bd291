mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cull.py -x -q -rf > gpurun_out/pytest_cull.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cull.log
( NAME=fp32 timeout 120 python tools/cull_micro.py
  NAME=tc RV_CULL_TC=1 timeout 120 python tools/cull_micro.py
  timeout 120 python tools/cull_ab.py run base
  RV_CULL_TC=1 timeout 120 python tools/cull_ab.py run base ) > gpurun_out/cull_ab8.log 2>&1
