mkdir -p gpurun_out
( timeout 300 python tools/cull_ab.py run base cv0 base cv0
  for v in base cv0; do
    if [ $v = base ]; then L=""; else L="RV_LIB=tools/bin/librotvote_$v.so"; fi
    env $L timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"cull_compact" --log-file gpurun_out/cv_$v.csv python tools/trace_cfg4.py > /dev/null 2>&1
  done ) > gpurun_out/cull_ab24.log 2>&1
