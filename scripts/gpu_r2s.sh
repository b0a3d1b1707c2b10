# round 2, pass s: per-op GEMM policy sweep at C2 shapes (G=16), one box
k() { env "$@" timeout 300 python scripts/kernel_bench.py --ops o,num,qkv,down --iters 30 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$*', d['op'], round(d['us'],1))"; }
for r in 1 2; do
k X=base
k ARMT_GEMM_PAIR=0
k ARMT_GEMM_PAIR=0 ARMT_GEMM_MC=0
k ARMT_GEMM_BN=128
k ARMT_GEMM_TMAE=0
k ARMT_GEMM_REM_CTAS=12
k ARMT_GEMM_REM_CTAS=28
done
