mkdir -p gpurun_out
RV_CULL_TC=1 timeout 120 python tools/cull_micro.py > gpurun_out/ct_plain.log 2>&1 && \
RV_CULL_TC=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cull_tc -s 8 -c 1 \
  -o gpurun_out/ct_l1_full -f python tools/cull_micro.py > gpurun_out/ct_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/ct_ncu.log
