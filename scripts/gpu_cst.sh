timeout 240 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -4 > gpurun_out/cst_t.log
grep -q passed gpurun_out/cst_t.log || exit 1
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/cst_t.log
rm -f gpurun_out/cst_sb.txt
for v in 0 1 0 1; do
  ARMT_GEMM_CST=$v timeout 200 python scripts/step_breakdown.py > gpurun_out/cst_sb_$v.log 2>&1
  echo "CST=$v" >> gpurun_out/cst_sb.txt; head -8 gpurun_out/cst_sb_$v.log >> gpurun_out/cst_sb.txt
done
