mkdir -p gpurun_out
( for v in a6 a22 a16; do NAME=$v RV_CULL_TC=1 RV_LIB=tools/bin/librotvote_$v.so timeout 120 python tools/cull_micro.py; done
  NAME=base timeout 120 python tools/cull_micro.py ) > gpurun_out/cull_ab22.log 2>&1
