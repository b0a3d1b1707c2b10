# round 2, pass an: three residual tiles in flight per warp in the TMA epilogue (no-split case)
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "tma or retrieve or fold" > gpurun_out/r2an_ktest.log 2>&1
tail -1 gpurun_out/r2an_ktest.log
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops num,foldtc --iters 50 | cut -c1-70 | sed "s/^/new /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_tmae2.so timeout 300 python scripts/kernel_bench.py --ops num,foldtc --iters 50 | cut -c1-70 | sed "s/^/old /"
done
