# round 2, pass v: packed-f32x2 SwiGLU + one polling warp per epilogue warpgroup (A/B vs HEAD); attention spin-lock / poly A/B
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or swiglu" > gpurun_out/r2v_ktest.log 2>&1
tail -1 gpurun_out/r2v_ktest.log
k() { env "$@" timeout 300 python scripts/kernel_bench.py --ops gu,down,o,attn --iters 30 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$*', d['op'], round(d['us'],1))"; }
run() { env "$@" timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-sequential > gpurun_out/r2v_tmp.log 2>&1;
  python -c "import json;d=json.loads(open('gpurun_out/r2v_tmp.log').read().strip().splitlines()[-1]);print('$*', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))"; }
for r in 1 2; do
  k X=new
  k ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_head.so
done
for r in 1 2; do
  run X=new
  run ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_head.so
done
for v in mutexspin mutexspinpoly4 poly2 poly4; do
  ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_$v.so timeout 300 python scripts/kernel_bench.py --ops attn --iters 50 | sed "s/^/$v /"
done
