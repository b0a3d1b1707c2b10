# round 2, pass ak: three-softmax-group attention (ARMT_ATTN=3) - correctness, A/B
set -x
ARMT_ATTN=3 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > gpurun_out/r2ak_ktest.log 2>&1
tail -3 gpurun_out/r2ak_ktest.log
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/two /"
  ARMT_ATTN=3 timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/three /"
done
ARMT_ATTN=3 timeout 300 python scripts/kernel_bench.py --G 1 --ops attn --iters 50 | sed "s/^/three_G1 /"
timeout 300 python scripts/kernel_bench.py --G 1 --ops attn --iters 50 | sed "s/^/two_G1 /"
