mkdir -p gpurun_out
( for v in base abl1 abl2 abl3 s6 s10 p2 p6 i4 i16 l2; do
   if [ $v = base ]; then NAME=$v RV_CULL_TC=1 timeout 120 python tools/cull_micro.py; else NAME=$v RV_CULL_TC=1 RV_LIB=tools/bin/librotvote_$v.so timeout 120 python tools/cull_micro.py; fi
  done
  RV_CULL_TC=1 timeout 300 python tools/cull_ab.py run base s6 s10 p2 p6 i4 i16 l2 ) > gpurun_out/cull_ab9.log 2>&1
