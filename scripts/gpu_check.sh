set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python scripts/kernel_bench.py --G 16 > gpurun_out/kb.log 2>&1
timeout 600 python scripts/step_breakdown.py > gpurun_out/sb.log 2>&1
tail -3 gpurun_out/*.log
