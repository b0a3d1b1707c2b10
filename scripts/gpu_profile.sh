# Round profile evidence (run under gpurun; outputs in gpurun_out/, summarised into profiles/ by
# scripts/profile_summary.py):
#   1. launch list of a 24-segment C2 forward (eager warm pass + one graph replay)
#   2. one --set full capture per hot kernel (C2 shapes, 16 members = one full wavefront step)
set -x
NCU="ncu --clock-control none"
timeout 900 $NCU --metrics gpu__time_duration.sum -c 4000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 0 --segments 24 --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/full_gu_g8 \
  python scripts/kernel_bench.py --G 8 --ops gu --iters 1 > gpurun_out/full_gu_g8.log 2>&1
for op in gu down o num lm; do
  timeout 600 $NCU --set full --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/full_$op \
    python scripts/kernel_bench.py --G 16 --ops $op --iters 1 > gpurun_out/full_$op.log 2>&1
done
timeout 600 $NCU --set full --import-source on -k regex:gemm_kernel -s 6 -c 2 -o gpurun_out/full_qkv \
  python scripts/kernel_bench.py --G 16 --ops qkv --iters 1 > gpurun_out/full_qkv.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:attn -s 3 -c 1 -o gpurun_out/full_attn \
  python scripts/kernel_bench.py --G 16 --ops attn --iters 1 > gpurun_out/full_attn.log 2>&1
timeout 600 $NCU --set full --import-source on -k "regex:fold|gemm" -s 5 -c 5 -o gpurun_out/full_fold \
  python scripts/kernel_bench.py --G 16 --ops foldtc --iters 1 > gpurun_out/full_fold.log 2>&1
# summarise on the box (ncu -i), keep the summaries + the launch list, drop the big reports
python scripts/profile_summary.py --tag ${TAG:-r2} --out gpurun_out/profiles_new --launches gpurun_out/launches.csv \
  --note "Launch list: \`ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 python bench.py --steps 1 --warmup 0 --segments 24 --no-cpu-baseline\` (C2 width, 24 segments; eager warm pass + one graph replay; cold-cache, serialised launches - compare SHARES, not absolutes). Full captures: \`ncu --set full --import-source on --clock-control none\` of scripts/kernel_bench.py at C2 shapes, G=16 (one wavefront step) unless noted. Command script: scripts/gpu_profile.sh." \
  --full gemm_gu=gpurun_out/full_gu.ncu-rep --full gemm_gu_g8=gpurun_out/full_gu_g8.ncu-rep \
  --full gemm_down=gpurun_out/full_down.ncu-rep --full gemm_qkv_rope=gpurun_out/full_qkv.ncu-rep \
  --full gemm_o_residual=gpurun_out/full_o.ncu-rep --full gemm_num_retrieve=gpurun_out/full_num.ncu-rep \
  --full gemm_lm_head_pair=gpurun_out/full_lm.ncu-rep --full attention_pp=gpurun_out/full_attn.ncu-rep \
  --full fold=gpurun_out/full_fold.ncu-rep > gpurun_out/profile_summary.log 2>&1
mkdir -p gpurun_out/reps
mv gpurun_out/full_gu.ncu-rep gpurun_out/full_attn.ncu-rep gpurun_out/reps/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
gzip -f gpurun_out/launches.csv
