# round 2, pass l: attention A/B (v1 committed / v2 / v2 without cross-head tail items) + v2 timeline trace
set -x
for r in 1 2; do
  for v in attnv1 noxtail; do
    ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_$v.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/$v /"
  done
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/v2 /"
done
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_trace.so timeout 300 python scripts/attn_trace.py > gpurun_out/r2l_trace.log 2>&1
head -20 gpurun_out/r2l_trace.log
