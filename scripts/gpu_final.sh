# round-end style checks on one GPU: tests, smoke, default bench, other configs, sharded plumbing
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/fin_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/fin_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/fin_bench.log 2>&1
run() { tag=$1; shift; timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline "$@" > gpurun_out/fin_cfg_$tag.log 2>&1; }
run c5 --config c5
run c4 --config c4 --steps 1 --warmup 1
run c2_seq --config c2 --schedule sequential
ARMT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/fin_gloo2.log 2>&1
for f in gpurun_out/fin_bench.log gpurun_out/fin_cfg_*.log gpurun_out/fin_gloo2.log; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f, round(d["value"]), round(d["ms_per_step"], 1), round(d["e2e"]["value"]), d["e2e"].get("mean_nll"), d["clocks"]["sm_mhz"], (d.get("roofline") or {}).get("frac"))
except Exception as e:
    print(f, "FAILED", e)
PY
done > gpurun_out/fin_summary.txt
