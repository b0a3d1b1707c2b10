# round 2, pass z: bench.py under torchrun (2 ranks sharing one GPU, gloo) after the repeated-graph fix; sharded gpu tests
set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py -q > gpurun_out/r2z_tests.log 2>&1
tail -1 gpurun_out/r2z_tests.log
ARMT_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2z_tr2.log 2>&1
echo "torchrun rc=$?"
grep '^{' gpurun_out/r2z_tr2.log | tail -1
ARMT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29518 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/r2z_ref2.log 2>&1
echo "ref torchrun rc=$?"
grep '^{' gpurun_out/r2z_ref2.log | tail -1 | cut -c1-400
