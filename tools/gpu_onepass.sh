mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_onepass.py -x -q -rf > gpurun_out/onepass.log 2>&1; echo "rc=$?" >> gpurun_out/onepass.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
