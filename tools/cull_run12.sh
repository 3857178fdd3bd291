mkdir -p gpurun_out
( for v in spin a7s a5 a6; do NAME=$v RV_CULL_TC=1 RV_LIB=tools/bin/librotvote_$v.so timeout 120 python tools/cull_micro.py; done ) > gpurun_out/cull_ab12.log 2>&1
