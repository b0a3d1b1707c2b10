# round 2, pass e: fold v2 latency fixes; parity A/B v1/v2; attention poly-fraction A/B
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "fold" > gpurun_out/r2e_foldtest.log 2>&1
tail -2 gpurun_out/r2e_foldtest.log
timeout 300 python scripts/fold_ab_parity.py > gpurun_out/r2e_par.log 2>&1
ARMT_FOLD_V1=1 timeout 300 python scripts/fold_ab_parity.py >> gpurun_out/r2e_par.log 2>&1
cat gpurun_out/r2e_par.log | grep -v Warn
for r in 1 2; do
timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 | grep foldtc
ARMT_FOLD_V1=1 timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 | grep foldtc
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_fold_ncu.csv \
  python scripts/kernel_bench.py --ops foldtc --iters 1 > /dev/null 2>&1
for r in 1 2; do
for v in 0 1 2 4 8; do
  if [ $v = 0 ]; then L=""; else L=gpu_ab/libarmt_poly$v.so; fi
  ARMT_LIB_PATH=$PWD/$L timeout 300 python scripts/kernel_bench.py --ops attn --iters 30 | grep attn | sed "s/^/poly$v /"
done
done
