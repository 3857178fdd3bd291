# ncu --set full of the fused refinement (one cfg4 solve after warm-up)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refine1 -s 3 -c 1 \
  -o gpurun_out/prof_refine1 -f python tools/onepass_diag.py cfg4 > gpurun_out/ncu_refine1.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_refine1.log
