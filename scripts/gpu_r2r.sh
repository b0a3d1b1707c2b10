# round 2, pass r: fold prep 4x4 K blocks + GEMM-R / fold_w SM split - tests, timings, ncu of the fold kernels
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "fold" > gpurun_out/r2r_ktest.log 2>&1
tail -1 gpurun_out/r2r_ktest.log
for r in 1 2 3; do timeout 300 python scripts/kernel_bench.py --ops foldtc --iters 50; done
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:fold|gemm" -s 5 -c 5 -o gpurun_out/r2r_fold \
  python scripts/kernel_bench.py --G 16 --ops foldtc --iters 1 > gpurun_out/r2r_ncu.log 2>&1
ncu -i gpurun_out/r2r_fold.ncu-rep --page details --csv > gpurun_out/r2r_fold_details.csv 2>&1
python scripts/ncu_sass_stalls.py gpurun_out/r2r_fold.ncu-rep fold_w 30 > gpurun_out/r2r_foldw_sass.txt 2>&1
python scripts/ncu_srcprof.py gpurun_out/r2r_fold.ncu-rep fold_w 30 > gpurun_out/r2r_foldw_src.txt 2>&1
ncu -i gpurun_out/r2r_fold.ncu-rep --page raw --csv --metrics gpu__time_duration.sum 2>/dev/null | python -c "import csv,sys; r=list(csv.reader(sys.stdin)); h=r[0]; k=h.index(\"Kernel Name\"); v=h.index(\"gpu__time_duration.sum\"); [print(x[k][:50], x[v]) for x in r[2:]]"
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2r_parity.log 2>&1
tail -1 gpurun_out/r2r_parity.log
