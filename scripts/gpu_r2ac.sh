# round 2, pass ac: fold prep split only when the K blocks exceed the SM count - tests (incl. G=16), timings
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "fold" > gpurun_out/r2ac_ktest.log 2>&1
tail -1 gpurun_out/r2ac_ktest.log
for G in 16 8 1; do
  timeout 300 python scripts/kernel_bench.py --G $G --ops foldtc --iters 50 | sed "s/^/new /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_prevfold.so timeout 300 python scripts/kernel_bench.py --G $G --ops foldtc --iters 50 | sed "s/^/prev /"
done
