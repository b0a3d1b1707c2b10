# round 2, pass ah: attention next-item L2 prefetch / 5 K/V stages A/B (v1 structure)
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/base /"
  for v in pf nst5 pfnst5; do
    ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_$v.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/$v /"
  done
done
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_pfnst5.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -1
