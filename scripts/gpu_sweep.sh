# usage: bash scripts/gpu_sweep.sh  -- GPU tests + bench sweeps (outputs under gpurun_out/)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests.log
for f in ${SWEEP:-16}; do
  ARMT_LM_FREE_SMS=$f timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_free$f.log 2>&1
done
for f in gpurun_out/*.log; do echo "== $f"; tail -4 $f | cut -c1-600; done
