# round 2, pass aa: new sharded regression test; compute-sanitizer memcheck over C2 layer shapes (pairs, multicast, TMA epilogue, fold v2)
set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py -q > gpurun_out/r2aa_tests.log 2>&1
tail -1 gpurun_out/r2aa_tests.log
mkdir -p gpurun_out/sanitize
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py c2w \
  > gpurun_out/sanitize/memcheck_c2w.log 2>&1
echo "memcheck c2w rc=$? $(grep -h 'ERROR SUMMARY' gpurun_out/sanitize/memcheck_c2w.log | tail -1)"
timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize.py c2w \
  > gpurun_out/sanitize/synccheck_c2w.log 2>&1
echo "synccheck c2w rc=$? $(grep -h 'ERROR SUMMARY' gpurun_out/sanitize/synccheck_c2w.log | tail -1)"
