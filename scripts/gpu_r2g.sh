# round 2, pass g: fold audit on C1 (v1 vs v2), ncu full of the v2 fold kernels, SwiGLU epilogue A/B
set -x
timeout 600 python scripts/fold_audit.py --config c1 --segments 8 --eps 1.0 > gpurun_out/r2g_audit_c1_v2.log 2>&1
ARMT_FOLD_V1=1 timeout 600 python scripts/fold_audit.py --config c1 --segments 8 --eps 1.0 > gpurun_out/r2g_audit_c1_v1.log 2>&1
tail -1 gpurun_out/r2g_audit_c1_v2.log gpurun_out/r2g_audit_c1_v1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fold_ -c 3 -o gpurun_out/r2g_fold \
  python scripts/kernel_bench.py --ops foldtc --iters 1 > gpurun_out/r2g_ncu.log 2>&1
for r in 1 2; do
  timeout 300 python scripts/kernel_bench.py --ops gu,qkv --iters 30 | sed "s/^/fast /"
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_swiglu_ieee.so timeout 300 python scripts/kernel_bench.py --ops gu,qkv --iters 30 | sed "s/^/ieee /"
done
