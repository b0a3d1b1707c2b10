timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/dyn_t.log
rm -f gpurun_out/bench_ab.txt
for rep in 1 2; do
for cfg in "0 0" "0 1" "1 1"; do
  set -- $cfg
  ARMT_DUAL=$1 ARMT_GEMM_DYN=$2 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bab.log').read().strip().splitlines()[-1]);print('dual=$1 dyn=$2', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> gpurun_out/bench_ab.txt
done; done
