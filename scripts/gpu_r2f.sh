# round 2, pass f: fold v2 (blocked W solve, [hi|lo] memory operand) — tests, A/B, launch list, bench
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "fold or gemm" > gpurun_out/r2f_ktest.log 2>&1
tail -3 gpurun_out/r2f_ktest.log
timeout 300 python scripts/fold_ab_parity.py > gpurun_out/r2f_par.log 2>&1
ARMT_FOLD_V1=1 timeout 300 python scripts/fold_ab_parity.py >> gpurun_out/r2f_par.log 2>&1
grep -v Warn gpurun_out/r2f_par.log
for r in 1 2; do
timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 | grep foldtc
ARMT_FOLD_V1=1 timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 | grep foldtc
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_fold_ncu.csv \
  python scripts/kernel_bench.py --ops foldtc --iters 1 > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2f_tests.log 2>&1
tail -5 gpurun_out/r2f_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2f_bench.log 2>&1
tail -c 400 gpurun_out/r2f_bench.log
