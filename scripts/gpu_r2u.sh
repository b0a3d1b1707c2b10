# round 2, pass u: full gpu suite, smoke, default bench (with sequential + cpu baseline), kernel timings
set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2u_tests.log 2>&1
tail -3 gpurun_out/r2u_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2u_smoke.log 2>&1
tail -1 gpurun_out/r2u_smoke.log
timeout 900 python bench.py > gpurun_out/r2u_bench.log 2>&1
tail -1 gpurun_out/r2u_bench.log
timeout 600 python scripts/kernel_bench.py --iters 30 > gpurun_out/r2u_kbench.log 2>&1
cat gpurun_out/r2u_kbench.log
