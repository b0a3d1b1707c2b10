# round 2, pass aw: d_head-128 attention buffering A/B (2 Q buffers + 3 K/V stages vs 1 Q buffer + 4/5 stages)
set -x
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_qb1nst5.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k dh128 2>&1 | tail -1
for r in 1 2; do
  python scripts/attn128_bench.py 32 | cut -c1-60 | sed "s/^/qb2nst3 /"
  for v in qb1nst5 qb1nst4; do ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_$v.so python scripts/attn128_bench.py 32 | cut -c1-60 | sed "s/^/$v /"; done
done
