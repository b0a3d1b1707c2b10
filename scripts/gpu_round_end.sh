# round evidence in one call: profiles (summaries built on the box), every BASELINE config, tests, smoke
bash scripts/gpu_profile.sh > gpurun_out/profile_run.log 2>&1
bash scripts/gpu_configs.sh
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/re_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/re_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/re_bench.log 2>&1
rm -rf gpurun_out/reps
