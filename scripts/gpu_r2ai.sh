# round 2, pass ai: gate/up as CTA pairs (+ concurrent remainder) vs multicast clusters, whole forward under the power cap
run() { env "$@" timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-sequential > gpurun_out/r2ai_tmp.log 2>&1;
  python -c "import json;d=json.loads(open('gpurun_out/r2ai_tmp.log').read().strip().splitlines()[-1]);print('$*', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'), round(d['roofline']['frac'],3))"; }
for r in 1 2 3; do
  run X=base
  run ARMT_GEMM_PAIR=conc
done
k() { env "$@" timeout 300 python scripts/kernel_bench.py --ops gu --iters 30 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$*', d['op'], round(d['us'],1))"; }
k X=base
k ARMT_GEMM_PAIR=conc
