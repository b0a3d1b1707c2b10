# A/B of GEMM pair modes in situ (step_breakdown per-op sums) and kernel_bench, same box
for v in 0 1 conc; do
  ARMT_GEMM_PAIR=$v timeout 600 python scripts/step_breakdown.py > gpurun_out/sb_$v.log 2>&1
done
for v in 0 conc; do
  ARMT_GEMM_PAIR=$v timeout 600 python scripts/step_breakdown.py > gpurun_out/sb2_$v.log 2>&1
done
ARMT_GEMM_PAIR=conc timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "pair or store" 2>&1 | tail -3 > gpurun_out/conc_t.log
