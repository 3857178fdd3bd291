mkdir -p gpurun_out
( for v in a3 a4 a7 a8 a11 a15; do NAME=$v RV_CULL_TC=1 RV_LIB=tools/bin/librotvote_$v.so timeout 120 python tools/cull_micro.py; done ) > gpurun_out/cull_ab11.log 2>&1
