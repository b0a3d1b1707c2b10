# A/B two builds of the library on one box: gpu_ab/libarmt_old.so (A) vs the in-tree build (B)
OLD=$PWD/gpu_ab/libarmt_old.so
for r in 1 2 3; do
  ARMT_LIB_PATH=$OLD timeout 300 python scripts/kernel_bench.py --ops gu,down,qkv,o,num,attn --iters 30 > gpurun_out/ab_k_old_$r.log 2>&1
  timeout 300 python scripts/kernel_bench.py --ops gu,down,qkv,o,num,attn --iters 30 > gpurun_out/ab_k_new_$r.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2 > gpurun_out/ab_tests.log
for r in 1 2; do
  ARMT_LIB_PATH=$OLD timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_b_old_$r.log 2>&1
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_b_new_$r.log 2>&1
done
