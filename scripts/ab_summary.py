"""Summarise scripts/gpu_lib_ab.sh output (gpurun_out/ab_*)."""
import collections
import glob
import json

k = collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/ab_k_*.log")):
    arm = f.split("_")[3]
    for line in open(f):
        try:
            r = json.loads(line)
        except ValueError:
            continue
        k[(r["op"], arm)].append(round(r["us"], 1))
for key, v in sorted(k.items()):
    print(key, v)
for f in sorted(glob.glob("gpurun_out/ab_b_*.log")):
    try:
        r = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(r["value"]), round(r["ms_per_step"], 1))
    except (ValueError, IndexError, KeyError):
        print(f, "ERR", open(f).read()[-300:])
print(open("gpurun_out/ab_tests.log").read())
