# round 2, pass bh: whole-forward A/B of the PDL and fused-DPFP switches on the final code
run() { env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-sequential > gpurun_out/r2bh_tmp.log 2>&1;
  python -c "import json;d=json.loads(open('gpurun_out/r2bh_tmp.log').read().strip().splitlines()[-1]);print('$*', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"; }
for r in 1 2; do
  run X=base
  run ARMT_PDL=0
  run ARMT_FUSED_DPFP=0
done
