"""Per-source-line warp-stall samples and executed instructions of one kernel in an
ncu report (cuda,sass view). python scripts/ncu_srcprof.py REPORT KERNEL_REGEX [TOP]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
data, fname, hdr = [], "", None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or len(r) < 8:
        continue
    try:
        data.append((float(r[4] or 0), float(r[7] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
    except ValueError:
        pass
ts = sum(d[0] for d in data) or 1
ti = sum(d[1] for d in data) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.0f}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{100 * d[0] / ts:5.1f}% smp {100 * d[1] / ti:5.1f}% ins  {d[2]:>18}  {d[3]}")
