mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cull.py -x -q -rf > gpurun_out/pytest_cull.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cull.log
( NAME=dyn timeout 120 python tools/cull_micro.py
  NAME=dyn0 RV_LIB=tools/bin/librotvote_dyn0.so timeout 120 python tools/cull_micro.py
  timeout 300 python tools/cull_ab.py run base dyn0 base dyn0 ) > gpurun_out/cull_ab25.log 2>&1
