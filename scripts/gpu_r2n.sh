# round 2, pass n: attention v4 (chunked item order for L2 reuse, L2 prefetch of the next item, 5 K/V stages) A/B
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > gpurun_out/r2n_ktest.log 2>&1
tail -1 gpurun_out/r2n_ktest.log
for r in 1 2; do
  for v in attnv1 noxtail nopf nochunk nst4; do
    ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_$v.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/$v /"
  done
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/v4 /"
done
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_trace.so timeout 300 python scripts/attn_trace.py > gpurun_out/r2n_trace.log 2>&1
head -12 gpurun_out/r2n_trace.log
