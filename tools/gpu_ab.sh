# A/B of side libraries built by tools/ab.py (names in $V): level-1 micro and cfg4 solve -> gpurun_out/
mkdir -p gpurun_out
timeout 900 python tools/ab.py run --micro $V > gpurun_out/ab_micro.log 2>&1
timeout 900 python tools/ab.py run $V > gpurun_out/ab_solve.log 2>&1
