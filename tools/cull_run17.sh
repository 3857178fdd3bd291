mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cull.py -x -q -rf > gpurun_out/pytest_cull.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cull.log
( NAME=tw2 timeout 120 python tools/cull_micro.py
  for v in tw0 tw1 tw3 tw2p6 a6; do NAME=$v RV_LIB=tools/bin/librotvote_$v.so timeout 120 python tools/cull_micro.py; done
  timeout 300 python tools/cull_ab.py run base tw0 tw1 tw3 tw2p6 ) > gpurun_out/cull_ab17.log 2>&1
