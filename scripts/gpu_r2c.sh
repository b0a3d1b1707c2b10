# round 2, pass c: state check after re-entry - gpu tests, smoke, bench (both arms)
set -x
nvidia-smi --query-gpu=name,clocks.sm,power.limit --format=csv > gpurun_out/r2c_smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2c_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2c_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2c_ref.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2c_tests.log 2>&1
tail -n 5 gpurun_out/r2c_tests.log
