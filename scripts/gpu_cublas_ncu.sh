# ncu full capture of cuBLAS's kernel for the gate/up and down GEMMs (library baseline next to ours)
for op in gu down; do
  timeout 600 ncu --set full --clock-control none -k regex:"gemm|Kernel|sm100|nvjet" -s 2 -c 1 -o gpurun_out/cublas_$op python scripts/cublas_probe.py $op > gpurun_out/cublas_ncu_$op.log 2>&1
  ncu -i gpurun_out/cublas_$op.ncu-rep --page raw --csv --print-units base > gpurun_out/cublas_${op}_raw.csv 2>&1
  rm -f gpurun_out/cublas_$op.ncu-rep
done
