"""Liveness of the C5 (LLaMA-3.1-8B-shaped) bench fixture: reference initializer
(armt/weights.py:98-138, seed 0, w_v_mem x 1/32, bf16 grid) at a given eps_assoc.

    python scripts/c5_liveness.py [--segments 8] [--eps 10000]

bf16 device runs of the diagonal schedule: the live memory vs an inert one
(W_k = 0: nothing is ever stored, every read guarded). Prints one JSON line per
segment: logits moved by the memory (relative Frobenius, first --cols vocab
columns) and the fraction of retrieval rows whose |phi.z| <= eps_assoc (guarded).
A memory that changes the logits by well over the bf16 parity tolerance (2e-2)
is live; a fully guarded one is not."""
import argparse
import json
import os
import sys
import time
from dataclasses import replace

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import bench  # noqa: E402
from c2_horizon_table import run_mode  # noqa: E402
from paper_2506_05229_b200 import ModelConfig, init_weights, round_to_bf16  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--segments", type=int, default=8)
    ap.add_argument("--cols", type=int, default=16384)
    ap.add_argument("--eps", type=float, default=bench.EPS_C5)
    args = ap.parse_args()
    cfg = ModelConfig(**bench.C5, eps_assoc=args.eps, seed=0)
    t = time.time()
    w = init_weights(cfg, dtype=np.float32)
    w = replace(w, w_v_mem=w.w_v_mem * np.float32(1 / 32)).map_arrays(round_to_bf16)
    print(json.dumps({"event": "init", "seconds": time.time() - t, "eps_assoc": args.eps}), flush=True)
    S, seg = args.segments, cfg.segment_size
    n = S * seg
    ids = torch.as_tensor(np.random.default_rng([0, n]).integers(0, cfg.vocab_size, n, dtype=np.int64)).cuda()
    guard: dict = {}
    live, _, dt_live = run_mode("bf16", w, w, cfg, ids, S, args.cols, guard)
    inert, _, _ = run_mode("bf16_inert", w, w, cfg, ids, S, args.cols)
    for s in range(S):
        a, b = live[s * seg:(s + 1) * seg].double(), inert[s * seg:(s + 1) * seg].double()
        print(json.dumps({"event": "segment", "segment": s, "live_vs_inert": float((a - b).norm() / b.norm()),
                          "finite": bool(torch.isfinite(live[s * seg:(s + 1) * seg]).all()),
                          "guarded_rows": float(np.mean(guard[s]))}), flush=True)
    print(json.dumps({"event": "done", "eps_assoc": args.eps, "seconds_live_run": dt_live}), flush=True)


if __name__ == "__main__":
    main()
