# round 2, pass h: fold v2.2 (merged chain, cp.async), TMA epilogue, SwiGLU fast path — tests, A/B, bench
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/r2h_ktest.log 2>&1
tail -3 gpurun_out/r2h_ktest.log
for r in 1 2; do
timeout 300 python scripts/kernel_bench.py --ops foldtc,num,o --iters 50 | sed "s/^/tmae /"
ARMT_GEMM_TMAE=0 timeout 300 python scripts/kernel_bench.py --ops foldtc,num,o --iters 50 | sed "s/^/regs /"
done
ARMT_FOLD_V1=1 ARMT_GEMM_TMAE=0 timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 | sed "s/^/v1 /"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_fold_ncu.csv \
  python scripts/kernel_bench.py --ops foldtc --iters 1 > /dev/null 2>&1
timeout 600 python scripts/c1_seed_spread.py > gpurun_out/r2h_seed_v2.log 2>&1
ARMT_FOLD_V1=1 timeout 600 python scripts/c1_seed_spread.py > gpurun_out/r2h_seed_v1.log 2>&1
grep median gpurun_out/r2h_seed_v2.log gpurun_out/r2h_seed_v1.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2h_tests.log 2>&1
tail -4 gpurun_out/r2h_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2h_bench.log 2>&1
tail -c 300 gpurun_out/r2h_bench.log
