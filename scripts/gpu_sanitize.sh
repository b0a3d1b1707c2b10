# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize.py
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/sanitize
for cfg in c1 mid c2w; do
  for tool in memcheck racecheck synccheck; do
    timeout 1200 $CS --tool $tool --print-limit 20 python scripts/sanitize.py $cfg \
      > gpurun_out/sanitize/${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/sanitize/${tool}_${cfg}.log | tail -1)" \
      >> gpurun_out/sanitize/summary.txt
  done
done
cat gpurun_out/sanitize/summary.txt
