# round 2, pass b: per-layer A error by precision mode at full depth; sharded + parity gpu tests after the ADVICE fixes
set -x
timeout 900 python scripts/c2_depth_modes.py > gpurun_out/r2b_depth.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not full_depth" > gpurun_out/r2b_tests.log 2>&1
tail -n 5 gpurun_out/r2b_tests.log
