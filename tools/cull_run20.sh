mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cull.py -x -q -rf > gpurun_out/pytest_cull.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cull.log
( NAME=el1 timeout 120 python tools/cull_micro.py
  NAME=el0 RV_LIB=tools/bin/librotvote_el0.so timeout 120 python tools/cull_micro.py
  timeout 300 python tools/cull_ab.py run base el0 base el0 ) > gpurun_out/cull_ab20.log 2>&1
