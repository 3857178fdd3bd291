mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_onepass.py tests/test_gpu_multi.py tests/test_gpu_cull.py tests/test_gpu_dplan.py -x -q -rf > gpurun_out/t1.log 2>&1; echo "rc=$?" >> gpurun_out/t1.log
timeout 300 python tools/onepass_diag.py > gpurun_out/diag1.log 2>&1; echo "rc=$?" >> gpurun_out/diag1.log
