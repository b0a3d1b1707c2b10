# round 2, pass m: attention v3 (dependency-driven MMA issue) tests, A/B vs v1, timeline trace
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > gpurun_out/r2m_ktest.log 2>&1
tail -3 gpurun_out/r2m_ktest.log
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_noxtail.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention_dh64 > gpurun_out/r2m_ktest_noxtail.log 2>&1
tail -1 gpurun_out/r2m_ktest_noxtail.log
for r in 1 2; do
  for v in attnv1 noxtail; do
    ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_$v.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/$v /"
  done
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/v3 /"
done
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_trace.so timeout 300 python scripts/attn_trace.py > gpurun_out/r2m_trace.log 2>&1
head -20 gpurun_out/r2m_trace.log
