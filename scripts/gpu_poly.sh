rm -f gpurun_out/poly.txt
for v in base poly base poly; do
  if [ $v = poly ]; then export ARMT_LIB_PATH=$PWD/paper_2506_05229_b200/libarmt_b200_poly.so; else unset ARMT_LIB_PATH; fi
  echo "$v $(timeout 120 python scripts/kernel_bench.py --ops attn --iters 30 2>&1 | tail -1)" >> gpurun_out/poly.txt
done
export ARMT_LIB_PATH=$PWD/paper_2506_05229_b200/libarmt_b200_poly.so
timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -2 >> gpurun_out/poly.txt
