# round 2, pass ao: TMA epilogue refill issued one chunk later (A/B)
set -x
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_laterefill.so timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "tma or retrieve or fold" > gpurun_out/r2ao_ktest.log 2>&1
tail -1 gpurun_out/r2ao_ktest.log
for r in 1 2 3; do
  timeout 300 python scripts/kernel_bench.py --ops num,foldtc,o --iters 50 | cut -c1-60 | sed "s/^/base /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_laterefill.so timeout 300 python scripts/kernel_bench.py --ops num,foldtc,o --iters 50 | cut -c1-60 | sed "s/^/late /"
done
