# round 2, pass ag: dual-stream wavefront A/B on the current code (whole forward, same box)
run() { env "$@" timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-sequential > gpurun_out/r2ag_tmp.log 2>&1;
  python -c "import json;d=json.loads(open('gpurun_out/r2ag_tmp.log').read().strip().splitlines()[-1]);print('$*', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'), round(d['roofline']['frac'],3))"; }
for r in 1 2; do
  run X=base
  run ARMT_DUAL=1
done
