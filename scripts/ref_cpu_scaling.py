"""The reference's own CPU path (baseline/_ref, numba kernels, WorkerPool over all
host threads) at the C2 width for G = 1, 2, 4, 8, 16 members per step (SURVEY
§8(d)): one stacked retrieve -> forward -> update step per G on a short segment,
extrapolated by FLOPs to a full C2 cell, plus the C2 forward time each G implies
for the sequential (G = 1 for all 2,048 cells) and diagonal (G = 16 for the full
steps) schedules. One JSON line per G, then a summary line.

    python scripts/ref_cpu_scaling.py [--seg 32] [--reps 2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2506_05229_b200 import ModelConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seg", type=int, default=32)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    cfg = ModelConfig(**bench.C2, eps_assoc=bench.EPS_ASSOC, seed=0)
    S, L = 128, cfg.n_layers
    rates = {}
    for G in (1, 2, 4, 8, 16):
        t0 = time.time()
        rc = bench.ReferenceCells(bench.C2, bench.EPS_ASSOC, seg=args.seg, members=G)
        rc.step()   # warm-up (numba compile, first touch)
        best = min(rc.step()[0] for _ in range(args.reps))
        rate = G * bench.cell_flops(rc.cfg) / best
        rates[G] = rate
        print(json.dumps({"G": G, "cores": rc.cores, "cpu": bench.cpu_model(), "step_s": best,
                          "cell_gflops": rate / 1e9, "c2_cell_s": bench.cell_flops(cfg) / rate,
                          "setup_s": time.time() - t0}), flush=True)
    # C2 forward on the reference CPU path (cells only; the LM head is the same in both)
    seq_s = S * L * bench.cell_flops(cfg) / rates[1]
    diag_s = S * L * bench.cell_flops(cfg) / rates[16]
    print(json.dumps({"summary": "C2 cells, reference CPU path", "sequential_s": seq_s, "diagonal_full_group_s": diag_s,
                      "diag_over_seq": seq_s / diag_s}), flush=True)


if __name__ == "__main__":
    main()
