# A/B of GEMM variants at locked (base) clocks: per-launch durations from ncu.
# usage: ABVAR=ARMT_GEMM_PF ABVALS="0 4 8" OPS=gu,down bash scripts/gpu_ncu_ab.sh
for v in ${ABVALS:-0 1}; do
  env ${ABVAR:-ARMT_GEMM_PAIR}=$v timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:gemm_kernel --csv \
     python scripts/kernel_bench.py --ops ${OPS:-gu,down,qkv,lm} --iters 2 > gpurun_out/ncu_ab_$v.csv 2>/dev/null
done
