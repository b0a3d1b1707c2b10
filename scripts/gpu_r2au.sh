# round 2, pass au: BN=128 TMA epilogue with three residual tiles (two mainloop stages) - fold GEMM3
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "tma or retrieve or fold" > gpurun_out/r2au_ktest.log 2>&1
tail -1 gpurun_out/r2au_ktest.log
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops foldtc,num --iters 50 | cut -c1-60 | sed "s/^/ew3 /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_ew2.so timeout 300 python scripts/kernel_bench.py --ops foldtc,num --iters 50 | cut -c1-60 | sed "s/^/ew2 /"
done
timeout 300 python scripts/kernel_bench.py --G 1 --ops foldtc --iters 50 | cut -c1-60 | sed "s/^/ew3_G1 /"
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_ew2.so timeout 300 python scripts/kernel_bench.py --G 1 --ops foldtc --iters 50 | cut -c1-60 | sed "s/^/ew2_G1 /"
