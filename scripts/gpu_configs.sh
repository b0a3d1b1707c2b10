# every BASELINE config through bench.py (diagonal; sequential where the paper compares)
run() { tag=$1; shift; timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline "$@" > gpurun_out/cfg_$tag.log 2>&1; }
run c2 --config c2
run c2_seq --config c2 --schedule sequential
run c3_512 --config c3-512
run c3_512_seq --config c3-512 --schedule sequential
run c3_2048 --config c3-2048
run c3_2048_seq --config c3-2048 --schedule sequential
run c3_32k --config c3-32k
run c3_32k_seq --config c3-32k --schedule sequential
run c4 --config c4 --steps 2 --warmup 1
run c5 --config c5 --steps 2 --warmup 1
for f in gpurun_out/cfg_*.log; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    print(f, round(d["value"]), round(d["ms_per_step"], 1), round(d["e2e"]["value"]), d.get("whole_step_frac_of_sustained"), d["clocks"]["sm_mhz"])
except Exception as e:
    print(f, "FAILED", e)
PY
done > gpurun_out/cfg_summary.txt
