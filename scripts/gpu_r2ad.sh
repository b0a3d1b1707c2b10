# round 2, pass ad: attention with alternating slot direction per query-pair round (L2 reuse of K/V)
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > gpurun_out/r2ad_ktest.log 2>&1
tail -1 gpurun_out/r2ad_ktest.log
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/snake /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_nosnake.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/plain /"
done
for v in snake nosnake; do
  L=""; [ $v = nosnake ] && L=$PWD/gpu_ab/libarmt_nosnake.so
  ARMT_LIB_PATH=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:attn_pp -s 3 -c 1 --csv \
    python scripts/kernel_bench.py --ops attn --iters 1 2>/dev/null | grep attn_pp | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
