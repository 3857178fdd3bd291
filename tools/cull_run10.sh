mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_cull.py -x -q -rf > gpurun_out/pytest_cull.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cull.log
( for v in base epq2 l2 i16 i32 abl3 abl1; do
   if [ $v = base ]; then NAME=$v RV_CULL_TC=1 timeout 120 python tools/cull_micro.py; else NAME=$v RV_CULL_TC=1 RV_LIB=tools/bin/librotvote_$v.so timeout 120 python tools/cull_micro.py; fi
  done
  RV_CULL_TC=1 timeout 300 python tools/cull_ab.py run base epq2 l2 i16 i32 ) > gpurun_out/cull_ab10.log 2>&1
