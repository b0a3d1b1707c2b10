ARMT_LM_OVERLAP=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_logits" 2>&1 | tail -30 > gpurun_out/t_overlap.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_logits" 2>&1 | tail -30 > gpurun_out/t_nooverlap.log
timeout 300 python scripts/kernel_bench.py --G 16 --ops o,down,num,foldtc,lm > gpurun_out/kb2.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pf.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/o_full python scripts/kernel_bench.py --G 16 --ops o --iters 1 > gpurun_out/ncu_o.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/down_full python scripts/kernel_bench.py --G 16 --ops down --iters 1 > gpurun_out/ncu_down.log 2>&1
