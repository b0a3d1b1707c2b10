# round 2, pass bd: register-epilogue residual rows prefetched into L2 during the mainloop (O / down) A/B
set -x
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_epipf.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "residual or pair" 2>&1 | tail -1
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops o,down --iters 30 | cut -c1-50 | sed "s/^/base /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_epipf.so timeout 300 python scripts/kernel_bench.py --ops o,down --iters 30 | cut -c1-50 | sed "s/^/pf /"
done
