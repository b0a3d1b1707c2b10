# round 2, pass ap: O-projection with the (three-deep) TMA epilogue vs the register epilogue
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops o --iters 50 | cut -c1-60 | sed "s/^/reg /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_tmaeo.so timeout 300 python scripts/kernel_bench.py --ops o --iters 50 | cut -c1-60 | sed "s/^/tma /"
done
