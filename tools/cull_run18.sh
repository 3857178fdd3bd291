mkdir -p gpurun_out
for v in base ps256 psa1 psa2 psa3; do
  if [ $v = base ]; then L=""; else L="RV_LIB=tools/bin/librotvote_$v.so"; fi
  env $L NAME=$v timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"cull_plan_small|cull_tc" --log-file gpurun_out/ps_$v.csv python tools/ps_micro.py > gpurun_out/ps_$v.log 2>&1
done
