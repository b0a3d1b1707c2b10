# round 2, pass o: profile evidence for r2 (launch list + ncu full of the hot kernels) and in-situ per-op breakdowns
set -x
TAG=r2 bash scripts/gpu_profile.sh > gpurun_out/profile_run.log 2>&1
tail -3 gpurun_out/profile_summary.log
timeout 900 python scripts/step_breakdown.py --segments 32 --schedule diagonal > gpurun_out/r2o_break_diag.log 2>&1
timeout 1200 python scripts/step_breakdown.py --segments 32 --schedule sequential > gpurun_out/r2o_break_seq.log 2>&1
tail -40 gpurun_out/r2o_break_diag.log
tail -40 gpurun_out/r2o_break_seq.log
