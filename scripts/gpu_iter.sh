# quick iteration: GPU tests, per-kernel timings, per-op breakdown of one C2 forward
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/gpu_tests.log
timeout 300 python scripts/kernel_bench.py --G 16 ${KB_OPS:+--ops $KB_OPS} > gpurun_out/kb.log 2>&1
timeout 600 python scripts/step_breakdown.py > gpurun_out/sb.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
