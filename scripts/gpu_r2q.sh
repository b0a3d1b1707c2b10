# round 2, pass q: whole-forward A/B of the residual-GEMM split policy (same box)
run() { env "$@" timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-sequential > gpurun_out/r2q_tmp.log 2>&1;
  python -c "import json;d=json.loads(open('gpurun_out/r2q_tmp.log').read().strip().splitlines()[-1]);print('$*', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))"; }
for rep in 1 2; do
  run X=base
  run ARMT_GEMM_CONC_O=0
  run ARMT_GEMM_REM_CTAS=16
  run ARMT_GEMM_REM_CTAS=24
  run ARMT_GEMM_TMAE=0
done
