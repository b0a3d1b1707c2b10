rm -f gpurun_out/attn_ab.txt
for v in 1 p 1 p; do
  ARMT_ATTN=$v timeout 120 python scripts/kernel_bench.py --ops attn --iters 20 >> gpurun_out/attn_ab.txt 2>&1
  ARMT_ATTN=$v timeout 200 python scripts/step_breakdown.py > gpurun_out/attn_sb_$v.log 2>&1
  echo "ATTN=$v $(head -1 gpurun_out/attn_sb_$v.log | cut -c1-40) $(grep armt_attention gpurun_out/attn_sb_$v.log)" >> gpurun_out/attn_ab.txt
done
