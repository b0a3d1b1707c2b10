# round 2, pass ab: fold prep split (phi-only prep + one-wave K kernel) - tests, A/B, GEMM3 TMA-epilogue A/B
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "fold" > gpurun_out/r2ab_ktest.log 2>&1
tail -1 gpurun_out/r2ab_ktest.log
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 | sed "s/^/new /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_prevfold.so timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 | sed "s/^/prev /"
  ARMT_GEMM_TMAE=0 timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50 | sed "s/^/new_tmae0 /"
done
timeout 300 python scripts/kernel_bench.py --G 1 --ops foldtc --iters 50 | sed "s/^/new_G1 /"
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_prevfold.so timeout 300 python scripts/kernel_bench.py --G 1 --ops foldtc --iters 50 | sed "s/^/prev_G1 /"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:fold|gemm" -c 6 --csv \
  python scripts/kernel_bench.py --G 16 --ops foldtc --iters 1 2>/dev/null | grep -E "fold|gemm" | awk -F'","' '{print $5, $NF}' | tail -6
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2ab_parity.log 2>&1
tail -1 gpurun_out/r2ab_parity.log
