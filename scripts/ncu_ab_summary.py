"""Summarise gpurun_out/ncu_ab_*.csv (scripts/gpu_ncu_ab.sh): mean duration and
tensor-pipe % per kernel name and variant."""
import collections, csv, glob, re, statistics, sys

for path in sorted(glob.glob("gpurun_out/ncu_ab_*.csv")):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        continue
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        per[int(r[ii])]["k"] = re.sub(r"\(CUtensor.*", "", r[ki])
    agg = collections.defaultdict(list)
    for i, m in per.items():
        agg[m["k"]].append((m.get("gpu__time_duration.sum", 0), m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)))
    for k, v in agg.items():
        print(f"{path[-8:-4]:>6} {k:45s} n={len(v):2d} us={statistics.mean(x[0] for x in v)/1e3:8.1f} tensor%={statistics.mean(x[1] for x in v):5.1f}")
