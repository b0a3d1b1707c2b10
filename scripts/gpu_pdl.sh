timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pdl.txt
grep -q " passed" gpurun_out/pdl.txt || exit 1
rm -f gpurun_out/bench_ab.txt
ABVAR=ARMT_PDL ABVALS="0 1" bash scripts/gpu_bench_ab.sh
cat gpurun_out/bench_ab.txt >> gpurun_out/pdl.txt
