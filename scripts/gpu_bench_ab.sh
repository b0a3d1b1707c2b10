# same-box A/B of whole-forward bench variants: ABVAR=NAME ABVALS="a b" bash scripts/gpu_bench_ab.sh
for rep in 1 2; do
for v in ${ABVALS:-0 1}; do
  env ${ABVAR:-ARMT_LM_OVERLAP}=$v timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bab_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bab_$v.log').read().strip().splitlines()[-1]);print('${ABVAR:-ARMT_LM_OVERLAP}=$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> gpurun_out/bench_ab.txt
done; done
