# round 2, pass y: gpu suite after the GEMM policy refactor; bench.py under torchrun (2 ranks sharing one GPU, gloo)
set -x
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2y_tests.log 2>&1
tail -2 gpurun_out/r2y_tests.log
ARMT_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2y_tr2.log 2>&1
echo "torchrun rc=$?"
tail -c 2500 gpurun_out/r2y_tr2.log
