mkdir -p gpurun_out
( for v in base s12 s6 p3 p6 i48 i64 ce4k l4; do
   if [ $v = base ]; then NAME=$v timeout 120 python tools/cull_micro.py; else NAME=$v RV_LIB=tools/bin/librotvote_$v.so timeout 120 python tools/cull_micro.py; fi
  done
  timeout 400 python tools/cull_ab.py run base s12 s6 p3 p6 i48 i64 ce4k l4 ) > gpurun_out/cull_ab23.log 2>&1
