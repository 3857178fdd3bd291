# Round-end pass on one GPU: the -m gpu suite, then tools/final_measure.sh, then the other bench lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash tools/final_measure.sh
for c in cfg1 cfg2 cfg3; do
  timeout 600 python bench.py --workload $c --steps 20 --warmup 3 > gpurun_out/bench_$c.log 2>&1
done
timeout 300 python bench.py --method alg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_alg1.log 2>&1
timeout 600 python bench.py --method rigid --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rigid.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1
