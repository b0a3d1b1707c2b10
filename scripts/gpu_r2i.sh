# round 2, pass i (re-entry): confirm the committed tree on hardware — tests, smoke, bench, fold/num/o kernel timings, sanitizer
set -x
mkdir -p gpurun_out/sanitize
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2i_gpu.txt
timeout 600 python scripts/kernel_bench.py --ops foldtc,num,o,gu,attn --iters 50 > gpurun_out/r2i_kbench.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2i_tests.log 2>&1
tail -4 gpurun_out/r2i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2i_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2i_bench.log 2>&1
tail -c 3000 gpurun_out/r2i_bench.log
CS=/usr/local/cuda/bin/compute-sanitizer
for cfg in c1 mid; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $tool --print-limit 20 python scripts/sanitize.py $cfg \
      > gpurun_out/sanitize/${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitize/${tool}_${cfg}.log | tail -1)" \
      >> gpurun_out/sanitize/summary.txt
  done
done
cat gpurun_out/sanitize/summary.txt
