# round 2, pass am: final-state check - gpu suite, smoke, default bench
set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2am_tests.log 2>&1
tail -2 gpurun_out/r2am_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2am_smoke.log 2>&1
tail -2 gpurun_out/r2am_smoke.log
timeout 1200 python bench.py > gpurun_out/r2am_bench.log 2>&1
tail -1 gpurun_out/r2am_bench.log | cut -c1-400
