# round 2, pass k: attention v2 (cross-item pipelined MMA issue, deferred O epilogue, cross-head tail items)
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > gpurun_out/r2k_ktest.log 2>&1
tail -3 gpurun_out/r2k_ktest.log
for r in 1 2 3; do timeout 300 python scripts/kernel_bench.py --ops attn --iters 50; done > gpurun_out/r2k_attn.log 2>&1
cat gpurun_out/r2k_attn.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_pp -s 3 -c 1 -o gpurun_out/r2k_attn \
  python scripts/kernel_bench.py --ops attn --iters 1 > gpurun_out/r2k_ncu.log 2>&1
python scripts/ncu_srcprof.py gpurun_out/r2k_attn.ncu-rep attn_pp 40 > gpurun_out/r2k_attn_src.txt 2>&1
ncu -i gpurun_out/r2k_attn.ncu-rep --page details > gpurun_out/r2k_attn_details.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2k_parity.log 2>&1
tail -3 gpurun_out/r2k_parity.log
