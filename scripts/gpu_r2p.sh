# round 2, pass p: attention with the per-sub-partition MUFU lock (v1 structure) - tests, A/B, poly fractions
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > gpurun_out/r2p_ktest.log 2>&1
tail -1 gpurun_out/r2p_ktest.log
for r in 1 2; do
  for v in nomutex mutexpoly2 mutexpoly4; do
    ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_$v.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/$v /"
  done
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/mutex /"
done
