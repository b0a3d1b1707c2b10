# round 2, pass d: fold v2 — kernel test, timing vs v1, launch-level ncu, full gpu tests, bench
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "fold" > gpurun_out/r2d_foldtest.log 2>&1
tail -3 gpurun_out/r2d_foldtest.log
timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 > gpurun_out/r2d_kb_v2.log 2>&1
ARMT_FOLD_V1=1 timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 > gpurun_out/r2d_kb_v1.log 2>&1
cat gpurun_out/r2d_kb_v2.log gpurun_out/r2d_kb_v1.log | grep foldtc
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_fold_ncu.csv \
  python scripts/kernel_bench.py --ops foldtc --iters 1 > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_tests.log 2>&1
tail -3 gpurun_out/r2d_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2d_bench.log 2>&1
tail -c 600 gpurun_out/r2d_bench.log
