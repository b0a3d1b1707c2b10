# round 2, pass at: remainder SMs per op (QKV / down / O) at the kernel level
k() { env "$@" timeout 300 python scripts/kernel_bench.py --ops qkv,down,o --iters 30 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$*', d['op'], round(d['us'],1))"; }
for r in 1 2; do
for v in 14 16 18 20 22 24; do k ARMT_GEMM_REM_CTAS=$v; done
done
