# round 2, pass bb: d_head-128 attention with grid-sized slot chunks (L2 reuse, exact balance) vs round-major order
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" 2>&1 | tail -1
for r in 1 2; do
  for G in 32 16; do
    python scripts/attn128_bench.py $G | cut -c1-60 | sed "s/^/chunk /"
    ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_nochunk128.so python scripts/attn128_bench.py $G | cut -c1-60 | sed "s/^/round /"
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:attn_pp128 -s 3 -c 1 --csv python scripts/attn128_bench.py 32 2>/dev/null | grep attn_pp128 | awk -F'","' '{print "chunk", $(NF-2), $NF}'
