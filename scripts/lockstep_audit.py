"""Where does the bf16 path leave the f32 path? (GPU diagnostic)

Runs the production bf16 engine and the f32 parity engine in lockstep over
the diagonal schedule of a C2-width fixture and, after every step, compares
per member: the retrieval guard decisions (|phi.z| <= eps rows that differ),
the residual stream after retrieval, after the block, and the memory state
after the fold. Prints one JSON line per (segment, layer) cell.

    python scripts/lockstep_audit.py [--segments 3] [--layers 16] [--vocab 4096]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from fixtures import cli_tokens, conditioned_weights  # noqa: E402
from paper_2506_05229_b200 import ModelConfig  # noqa: E402
from paper_2506_05229_b200.engine import Engine, MemoryState, prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import diagonal_plan, segment_input  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    nb = float(b.norm())
    return float((a - b).norm()) / nb if nb > 0 else float((a - b).norm())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--segments", type=int, default=3)
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--vocab", type=int, default=4096)
    ap.add_argument("--eps", type=float, default=100.0)
    args = ap.parse_args()
    cfg = ModelConfig(n_layers=args.layers, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024,
                      num_mem_tokens=128, d_mem=64, vocab_size=args.vocab, eps_assoc=args.eps, seed=0)
    w = conditioned_weights(cfg)
    S = args.segments
    tokens = cli_tokens(cfg, S * cfg.segment_size - 13, seed=2)
    segs, _ = segment_input(tokens, cfg)
    ids = torch.as_tensor(np.concatenate(segs)).cuda()
    plan = diagonal_plan(S, cfg.n_layers)
    pb, pf = prepare_weights(w, "bf16"), prepare_weights(w, "f32")
    eb, ef = Engine(pb, plan.max_members, plan.n_slots), Engine(pf, plan.max_members, plan.n_slots)
    sb, sf = MemoryState.fresh(cfg), MemoryState.fresh(cfg)
    sb.sync_shadow(pb)
    stream = torch.cuda.current_stream().cuda_stream
    seg, T = cfg.segment_size, cfg.tokens_per_segment
    eps = pf.eps_assoc
    for step in plan.steps:
        for s, slot in step.enters:
            eb.embed(ids[s * seg:(s + 1) * seg], slot, stream)
            ef.embed(ids[s * seg:(s + 1) * seg], slot, stream)
        G = len(step.layers)
        x_in_b = eb.xs[step.slots].clone()
        x_in_f = ef.xs[step.slots].clone()
        eb.retrieve(step.slots, step.layers, sb, stream)
        ef.retrieve(step.slots, step.layers, sf, stream)
        torch.cuda.synchronize()
        xr_b, xr_f = eb.xs[step.slots].clone(), ef.xs[step.slots].clone()
        den_b, den_f = eb.den[:G].clone(), ef.den[:G].clone()
        eb.forward(step.slots, step.layers, stream)
        ef.forward(step.slots, step.layers, stream)
        torch.cuda.synchronize()
        y_b, y_f = eb.xs[step.slots].clone(), ef.xs[step.slots].clone()
        eb.update(step.slots, step.layers, sb, stream)
        ef.update(step.slots, step.layers, sf, stream)
        torch.cuda.synchronize()
        for g, nd in enumerate(step.nodes):
            l = nd.layer
            gb, gf = den_b[g].abs() <= eps, den_f[g].abs() <= eps
            near = ((den_f[g].abs() - eps).abs() / eps < 0.02).sum().item()
            dret_b = xr_b[g] - x_in_b[g]
            dret_f = xr_f[g] - x_in_f[g]
            print(json.dumps({
                "segment": nd.segment, "layer": l,
                "x_in": rel(x_in_b[g], x_in_f[g]),
                "guard_flips": int((gb != gf).sum().item()), "rows_within_2pct_of_eps": int(near),
                "guarded_f32": int(gf.sum().item()),
                "retrieved_delta": rel(dret_b, dret_f),
                "den": rel(den_b[g], den_f[g]),
                "x_after_retrieve": rel(xr_b[g], xr_f[g]),
                "y_block": rel(y_b[g], y_f[g]),
                "y_mem_rows": rel(y_b[g, seg:], y_f[g, seg:]),
                "A": rel(sb.A[l], sf.A[l]), "z": rel(sb.z[l], sf.z[l]),
            }), flush=True)


if __name__ == "__main__":
    main()
