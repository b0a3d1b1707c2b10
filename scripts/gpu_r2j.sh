# round 2, pass j: MUFU probe, C1 bf16 seed spread (fold v1 vs v2), attention ncu (source), full gpu suite without -x
set -x
./scripts/probe_mufu > gpurun_out/r2j_mufu.log 2>&1
timeout 600 python scripts/c1_seed_spread.py > gpurun_out/r2j_seed_v2.log 2>&1
ARMT_FOLD_V1=1 timeout 600 python scripts/c1_seed_spread.py > gpurun_out/r2j_seed_v1.log 2>&1
grep median gpurun_out/r2j_seed_v2.log gpurun_out/r2j_seed_v1.log
for r in 1 2 3; do timeout 300 python scripts/kernel_bench.py --ops attn --iters 50; done > gpurun_out/r2j_attn.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_pp -s 3 -c 1 -o gpurun_out/r2j_attn \
  python scripts/kernel_bench.py --ops attn --iters 1 > gpurun_out/r2j_ncu.log 2>&1
python scripts/ncu_srcprof.py gpurun_out/r2j_attn.ncu-rep attn_pp 60 > gpurun_out/r2j_attn_src.txt 2>&1
ncu -i gpurun_out/r2j_attn.ncu-rep --page raw --csv > gpurun_out/r2j_attn_raw.csv 2>&1
ncu -i gpurun_out/r2j_attn.ncu-rep --page details > gpurun_out/r2j_attn_details.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2j_tests.log 2>&1
tail -8 gpurun_out/r2j_tests.log
