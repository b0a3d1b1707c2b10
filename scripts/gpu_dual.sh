timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/dual_t.log
rm -f gpurun_out/bench_ab.txt
ABVAR=ARMT_DUAL ABVALS="0 1" bash scripts/gpu_bench_ab.sh
