# round 2, pass t: O-projection without the TMA epilogue: remainder SM sweep, then whole-forward A/B
k() { env "$@" timeout 300 python scripts/kernel_bench.py --ops o,num --iters 30 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$*', d['op'], round(d['us'],1))"; }
run() { env "$@" timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-sequential > gpurun_out/r2t_tmp.log 2>&1;
  python -c "import json;d=json.loads(open('gpurun_out/r2t_tmp.log').read().strip().splitlines()[-1]);print('$*', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))"; }
for v in 20 24 28 32 36; do k ARMT_GEMM_REM_CTAS_O=$v; done
for r in 1 2; do
  run X=new
  run ARMT_GEMM_REM_CTAS_O=20
  run ARMT_GEMM_REM_CTAS_O=32
done
