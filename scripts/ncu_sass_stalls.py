"""Top SASS instructions by warp-stall samples with their dominant stall reasons
(ncu source page, sass view). python scripts/ncu_sass_stalls.py REPORT KERNEL_REGEX [TOP]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
idx = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
tot = {r: 0 for r in reasons}
for k, r in enumerate(rows):
    if not r or r[0] in ("Address", "Kernel Name") or len(r) < len(hdr):
        continue
    s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    st = {h: float(r[idx[h]] or 0) for h in reasons}
    for h in reasons:
        tot[h] += st[h]
    data.append((s, k, r[idx["Source"]].strip(), st))
T = sum(d[0] for d in data) or 1
print("total samples %.0f; by reason: %s" % (T, ", ".join(f"{h[6:]} {100*v/T:.1f}%" for h, v in sorted(tot.items(), key=lambda x: -x[1]) if v)))
for s, k, src, st in sorted(data, reverse=True)[:top]:
    why = ", ".join(f"{h[6:]} {int(v)}" for h, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{100*s/T:5.1f}%  #{k:5d}  {src[:60]:60s}  {why}")
