mkdir -p gpurun_out
( timeout 300 python tools/cull_ab.py run base bf1 bf2
  for v in base bf1 bf2; do
    if [ $v = base ]; then L=""; else L="RV_LIB=tools/bin/librotvote_$v.so"; fi
    env $L timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"rv_vote_tc_kernel" --log-file gpurun_out/bf_$v.csv python tools/trace_cfg4.py > /dev/null 2>&1
  done ) > gpurun_out/cull_ab19.log 2>&1
