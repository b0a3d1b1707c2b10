timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/v_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/v_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/v_bench.log 2>&1
timeout 600 python bench.py --config c5 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/v_c5.log 2>&1
ARMT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/v_gloo2.log 2>&1
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/v_ref.log 2>&1
for f in gpurun_out/v_bench.log gpurun_out/v_c5.log gpurun_out/v_gloo2.log gpurun_out/v_ref.log; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f, round(d["value"], 1), round(d["ms_per_step"], 1), round(d["e2e"]["value"], 1), d["e2e"].get("mean_nll"), (d.get("roofline") or {}).get("frac"), (d.get("clocks") or {}).get("sm_mhz"))
except Exception as e:
    print(f, "FAILED", e)
PY
done > gpurun_out/v_summary.txt
