timeout 200 python -m pytest tests/test_gpu_kernels.py -x -q -k attention 2>&1 | tail -4 > gpurun_out/tp.txt
for v in smem tmem smem tmem; do
  if [ $v = smem ]; then export ARMT_LIB_PATH=$PWD/paper_2506_05229_b200/libarmt_b200_smemp.so; else unset ARMT_LIB_PATH; fi
  echo "$v $(timeout 120 python scripts/kernel_bench.py --ops attn --iters 30 2>&1 | tail -1)" >> gpurun_out/tp.txt
done
