timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/xp_t.log
timeout 600 python scripts/kernel_bench.py --ops o,num,down --env ARMT_GEMM_XPOSE --flags 0,1,0,1 > gpurun_out/xp_kb.log 2>&1
for v in 0 1 0 1; do
  ARMT_GEMM_XPOSE=$v timeout 600 python scripts/step_breakdown.py > gpurun_out/xp_sb_$v.log 2>&1
  head -12 gpurun_out/xp_sb_$v.log | grep -E "total|residual|retrieve|fold" >> gpurun_out/xp_sb.txt
done
