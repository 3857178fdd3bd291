mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cull.py -x -q -rf > gpurun_out/pytest_cull.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cull.log
( for v in base t1 t4 t2p2; do
   if [ $v = base ]; then NAME=$v timeout 120 python tools/cull_micro.py; else NAME=$v RV_LIB=tools/bin/librotvote_$v.so timeout 120 python tools/cull_micro.py; fi
  done
  NAME=tc RV_CULL_TC=1 timeout 120 python tools/cull_micro.py
  timeout 300 python tools/cull_ab.py run base t1 t4 t2p2
  RV_CULL_TC=1 timeout 120 python tools/cull_ab.py run base ) > gpurun_out/cull_ab7.log 2>&1
