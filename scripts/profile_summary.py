"""Summarise ncu outputs into profiles/ (tracked evidence).

    python scripts/profile_summary.py --launches gpurun_out/launches.csv \
        --full gemm_gu=gpurun_out/gemm_gu.ncu-rep [--full attn=...] --tag r1

Writes profiles/<tag>_launches.md (per-kernel share of device time from the
cold-cache, serialised launch list) and profiles/<tag>_kernels.json + .md
(key metrics of each full capture: duration, DRAM bytes, tensor-pipe %, L2 %,
derived DRAM GB/s and % of measured HBM, issue %, registers). bench.py reads the gate/up GEMM's DRAM bytes
from profiles/*_kernels.json as its roofline `traffic`.
"""

import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                            "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
}


def short(name: str) -> str:
    name = re.sub(r"\(CUtensorMap_st.*|\(ArmtMembers.*|\(const .*", "", name)
    name = name.replace("void ", "").replace("armt::", "")
    return name[:80]


def launches(path):
    text = open(path).read()
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        v *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += v
    return agg


def full_metrics(rep):
    """Key metrics of every kernel in a --set full report (one dict per launch)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res_all = []
    for v in rows[2:] if len(rows) > 2 else rows[1:]:
        if len(v) != len(h):
            continue
        res = {"kernel": short(v[h.index("Kernel Name")]) if "Kernel Name" in h else ""}
        for key, names in METRICS.items():
            m = next((n for n in ((names,) if isinstance(names, str) else names) if n in h), None)
            if m is not None:
                try:
                    res[key] = float(v[h.index(m)].replace(",", ""))
                except ValueError:
                    res[key] = v[h.index(m)]
        res_all.append(res)
    return res_all


def write_kernels_md(res, out_dir, tag, note):
    """DRAM GB/s is derived (bytes / duration) and set against the measured
    copy bandwidth in MEASURED_PEAKS.json, so the column never depends on
    which throughput-percentage name this ncu version exports."""
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm = json.load(open(peaks_path)).get("hbm_gbs") if os.path.exists(peaks_path) else None
    lines = [f"# {tag}: ncu --set full captures (one launch each)", "", note, "",
             f"DRAM GB/s = (dram__bytes_read.sum + dram__bytes_write.sum) / gpu__time_duration.sum; "
             f"% HBM is against the measured copy bandwidth ({hbm} GB/s, MEASURED_PEAKS.json).", "",
             "| capture | kernel | us | DRAM MB (r+w) | DRAM GB/s | % HBM | tensor % | L2 % | issue % | regs |",
             "|---|---|---:|---:|---:|---:|---:|---:|---:|---:|"]
    for label, m in res.items():
        dram = (m.get("dram_read_bytes", 0) + m.get("dram_write_bytes", 0)) / 1e6
        ns = m.get("duration_ns", 0)
        gbs = dram * 1e6 / ns if ns else 0.0
        pct = f"{gbs / hbm * 100:.1f}" if hbm else "-"
        lines.append(f"| {label} | `{m.get('kernel', '')}` | {ns / 1e3:.1f} | {dram:.1f} | {gbs:.0f} | {pct} | "
                     f"{m.get('tensor_pipe_pct', 0):.1f} | {m.get('l2_throughput_pct', 0):.1f} | "
                     f"{m.get('issue_active_pct', 0):.1f} | {m.get('registers', 0):.0f} |")
    open(os.path.join(out_dir, f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full", action="append", default=[])
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--note", default="")
    ap.add_argument("--from-json", help="rewrite <tag>_kernels.md from an existing <tag>_kernels.json")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    if args.launches:
        agg = launches(args.launches)
        tot = sum(v[1] for v in agg.values())
        lines = [f"# {args.tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
                 args.note, "", f"total device time in capture: {tot / 1e6:.3f} ms", "",
                 "| share | total ms | launches | avg us | kernel |", "|---:|---:|---:|---:|---|"]
        for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| {v / tot * 100:.1f}% | {v / 1e6:.3f} | {n} | {v / n / 1e3:.1f} | `{k}` |")
        open(os.path.join(args.out, f"{args.tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    if args.full:
        res = {}
        for item in args.full:
            label, rep = item.split("=", 1)
            for k, m in enumerate(full_metrics(rep)):
                res[label if k == 0 else f"{label}.{k}"] = m
        json.dump(res, open(os.path.join(args.out, f"{args.tag}_kernels.json"), "w"), indent=1)
        write_kernels_md(res, args.out, args.tag, args.note)
    if args.from_json:
        res = json.load(open(args.from_json))
        write_kernels_md(res, args.out, args.tag, args.note)


if __name__ == "__main__":
    main()
