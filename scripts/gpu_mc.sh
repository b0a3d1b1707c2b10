# short per-command timeouts: a hung kernel must not eat the call
timeout 240 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -6 > gpurun_out/mc_t.log || exit 1
grep -q passed gpurun_out/mc_t.log || exit 1
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 >> gpurun_out/mc_t.log
timeout 120 python scripts/kernel_bench.py --ops attn --iters 20 > gpurun_out/mc_attn.log 2>&1
rm -f gpurun_out/mc_sb.txt
for v in 0 1 0 1; do
  ARMT_GEMM_MC=$v timeout 200 python scripts/step_breakdown.py > gpurun_out/mc_sb_$v.log 2>&1
  echo "MC=$v" >> gpurun_out/mc_sb.txt; head -10 gpurun_out/mc_sb_$v.log >> gpurun_out/mc_sb.txt
done
