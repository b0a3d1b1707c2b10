# round 2, pass ay: the 64-key-step ping-pong kernel at d_head 64 (A/B vs the 128-key-step production kernel)
set -x
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_pp64.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_dh64 or attention_matches" 2>&1 | tail -1
for r in 1 2; do
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | cut -c1-60 | sed "s/^/prod /"
  for v in pp64 pp64nst6 pp64qb2; do ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_$v.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | cut -c1-60 | sed "s/^/$v /"; done
done
