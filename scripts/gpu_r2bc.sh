# round 2, pass bc: d_head-64 attention with grid-sized slot chunks vs the alternating-direction order
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -1
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | cut -c1-60 | sed "s/^/chunk /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_snakeonly.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | cut -c1-60 | sed "s/^/snake /"
done
timeout 300 python scripts/kernel_bench.py --G 1 --ops attn --iters 50 | cut -c1-60 | sed "s/^/chunk_G1 /"
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_snakeonly.so timeout 300 python scripts/kernel_bench.py --G 1 --ops attn --iters 50 | cut -c1-60 | sed "s/^/snake_G1 /"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:attn_pp -s 3 -c 1 --csv python scripts/kernel_bench.py --ops attn --iters 1 2>/dev/null | grep attn_pp | awk -F'","' '{print "chunk", $(NF-2), $NF}'
