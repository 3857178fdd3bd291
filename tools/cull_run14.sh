mkdir -p gpurun_out
( timeout 300 python tools/cull_ab.py run base ce512 ce1k ce2k ce4k
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ce2k.csv env RV_LIB=tools/bin/librotvote_ce2k.so python tools/trace_cfg4.py > /dev/null 2>&1; echo ncu rc=$? ) > gpurun_out/cull_ab14.log 2>&1
