# round 2, pass al: streaming (evict-first) stores for the logits, whole-forward A/B (same box) + sequential ratio
run() { env "$@" timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-sequential > gpurun_out/r2al_tmp.log 2>&1;
  python -c "import json;d=json.loads(open('gpurun_out/r2al_tmp.log').read().strip().splitlines()[-1]);print('$*', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'), round(d['roofline']['frac'],3))"; }
for r in 1 2 3; do
  run X=stream
  run ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_nostream.so
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  python bench.py --steps 1 --warmup 0 --segments 24 --no-cpu-baseline --no-sequential 2>/dev/null > gpurun_out/r2al_ncu_stream.csv
ARMT_LIB_PATH=$PWD/gpu_ab/libarmt_nostream.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  python bench.py --steps 1 --warmup 0 --segments 24 --no-cpu-baseline --no-sequential 2>/dev/null > gpurun_out/r2al_ncu_plain.csv
for f in stream plain; do python - gpurun_out/r2al_ncu_$f.csv $f <<'PY'
import csv, sys, collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h=rows[0]; k=h.index("Kernel Name"); mn=h.index("Metric Name"); mv=h.index("Metric Value")
tot=collections.defaultdict(float)
for r in rows[1:]:
    try: tot[r[mn]] += float(r[mv].replace(",",""))
    except ValueError: pass
print(sys.argv[2], {m: round(v/1e6, 1) for m, v in tot.items()})
PY
done
