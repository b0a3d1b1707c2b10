# Round profile evidence (run under gpurun; outputs in gpurun_out/, summarised into profiles/ by
# scripts/profile_summary.py):
#   1. launch list of a 24-segment C2 forward (eager warm pass + one graph replay)
#   2. one --set full capture per hot kernel (C2 shapes, 16 members = one full wavefront step)
set -x
NCU="ncu --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum -c 4000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 0 --segments 24 --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1
for op in gu down o num lm; do
  timeout 600 $NCU --set full --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/full_$op \
    python scripts/kernel_bench.py --G 16 --ops $op --iters 1 > gpurun_out/full_$op.log 2>&1
done
timeout 600 $NCU --set full --import-source on -k regex:gemm_kernel -s 6 -c 2 -o gpurun_out/full_qkv \
  python scripts/kernel_bench.py --G 16 --ops qkv --iters 1 > gpurun_out/full_qkv.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:attn -s 3 -c 1 -o gpurun_out/full_attn \
  python scripts/kernel_bench.py --G 16 --ops attn --iters 1 > gpurun_out/full_attn.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:fold -s 3 -c 3 -o gpurun_out/full_fold \
  python scripts/kernel_bench.py --G 16 --ops foldtc --iters 1 > gpurun_out/full_fold.log 2>&1
