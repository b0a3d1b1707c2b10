# round-2 first pass: full-depth parity tests, smoke (d_head 64), horizon table, bench with sequential
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_depth" --durations=5 > gpurun_out/r2a_tests.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2a_smoke.log 2>&1
timeout 1800 python scripts/c2_horizon_table.py > gpurun_out/r2a_horizon.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a_bench.log 2>&1
tail -5 gpurun_out/r2a_*.log
