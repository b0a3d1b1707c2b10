# round 2, pass av: d_head-128 ping-pong attention - tests, timing vs single-tile kernel and SDPA
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > gpurun_out/r2av_ktest.log 2>&1
tail -3 gpurun_out/r2av_ktest.log
python scripts/attn128_bench.py 16; python scripts/attn128_bench.py 32
ARMT_ATTN=tc python scripts/attn128_bench.py 32
