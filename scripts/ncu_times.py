"""Print (kernel, duration us) from `ncu --metrics gpu__time_duration.sum --csv --print-units base` on stdin."""
import csv
import re
import sys

rows = [r for r in csv.reader(sys.stdin) if len(r) > 5]
h = next(r for r in rows if r[0] == "ID")
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
for r in rows:
    if r is h or r[0] == "ID":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")[:60]
    print(f"{float(r[vi].replace(',', '')) / 1e3:10.1f} us  {name}")
