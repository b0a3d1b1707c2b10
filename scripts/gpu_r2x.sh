# round 2, pass x: C5 on the reference initializer - liveness at eps 1e4 / 3e3, bench line
set -x
free -g | head -2
timeout 1800 python scripts/c5_liveness.py --segments 8 --eps 10000 > gpurun_out/r2x_c5_live_1e4.log 2>&1
tail -12 gpurun_out/r2x_c5_live_1e4.log
timeout 1800 python scripts/c5_liveness.py --segments 8 --eps 3000 > gpurun_out/r2x_c5_live_3e3.log 2>&1
tail -12 gpurun_out/r2x_c5_live_3e3.log
timeout 1800 python bench.py --config c5 --init reference --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2x_c5_bench.log 2>&1
tail -c 1500 gpurun_out/r2x_c5_bench.log
