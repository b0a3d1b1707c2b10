timeout 240 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2 > gpurun_out/rpf.txt
for v in old new old new; do
  if [ $v = old ]; then export ARMT_LIB_PATH=$PWD/paper_2506_05229_b200/libarmt_b200_old.so; else unset ARMT_LIB_PATH; fi
  timeout 200 python scripts/step_breakdown.py > gpurun_out/rpf_sb.log 2>&1
  echo "$v $(head -1 gpurun_out/rpf_sb.log | cut -c1-30) $(grep -E 'residual_N2048_K2048|retrieve|fold_tc|K8192' gpurun_out/rpf_sb.log | awk '{print $1, $NF}' | tr '\n' ' ')" >> gpurun_out/rpf.txt
done
