timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -15 > gpurun_out/pair_tests.log
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 >> gpurun_out/pair_tests.log
timeout 600 python scripts/kernel_bench.py --ops gu,down,qkv,o,num,lm --flags 0,1 --repeat 2 > gpurun_out/pair_ab.log 2>&1
