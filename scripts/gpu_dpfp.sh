timeout 240 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -8 > gpurun_out/dpfp_t.log
grep -q " passed" gpurun_out/dpfp_t.log || exit 1
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/dpfp_t.log
rm -f gpurun_out/dpfp_sb.txt
for v in 0 1 0 1; do
  ARMT_FUSED_DPFP=$v timeout 200 python scripts/step_breakdown.py > gpurun_out/dpfp_sb_$v.log 2>&1
  echo "DPFP=$v" >> gpurun_out/dpfp_sb.txt; grep -E "total|N64|dpfp|retrieve" gpurun_out/dpfp_sb_$v.log >> gpurun_out/dpfp_sb.txt
done
