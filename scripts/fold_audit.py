"""Audit the tensor-core fold on the inputs it actually sees (GPU).

Runs the production bf16 path eagerly over the full-depth C2 fixture
(tests/test_gpu_parity.py::c2_full_depth) and, at every (segment, layer)
fold, replays the same k/v/beta projections and prior (A, z) through the
in-order f64 delta rule (armt/memory.py:94-125) on the host. Prints, per
cell, the relative error of the device A and z against that replay and the
smallest guard margins (|zq| - eps, nrm - eps, relative to eps) so guard
flips are visible.

    python scripts/fold_audit.py [--segments 3] [--layers 16] [--f32]
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


def dpfp(x, nu):
    r = np.concatenate([np.maximum(x, 0), np.maximum(-x, 0)], axis=-1)
    return np.concatenate([r * np.roll(r, -j, axis=-1) for j in range(1, nu + 1)], axis=-1)


def fold64(A, z, k, v, b, nu, eps):
    A = A.astype(np.float64).copy()
    z = z.astype(np.float64).copy()
    beta = 1.0 / (1.0 + np.exp(-b.astype(np.float64)))
    phi = dpfp(k.astype(np.float64), nu)
    zq_m, nrm_m = np.inf, np.inf
    for i in range(k.shape[0]):
        p = phi[i]
        zq = float(z @ p)
        nrm = float(p @ p)
        zq_m = min(zq_m, abs(abs(zq) - eps) / eps)
        nrm_m = min(nrm_m, abs(nrm - eps) / eps)
        vbar = np.zeros(A.shape[0]) if abs(zq) <= eps else (A @ p) / zq
        gamma = 0.0 if nrm <= eps else 1.0 - zq / nrm
        A += np.outer(beta[i] * (v[i].astype(np.float64) - vbar), p)
        z += gamma * p
    return A, z, zq_m, nrm_m


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--segments", type=int, default=3)
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--eps", type=float, default=100.0)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--config", default="c2", choices=["c2", "c1", "mid"])
    args = ap.parse_args()
    if args.config == "c2":
        cfg = ModelConfig(n_layers=args.layers, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024,
                          num_mem_tokens=128, d_mem=64, vocab_size=4096, eps_assoc=args.eps, seed=0)
    else:
        from conftest import C1, MID
        cfg = ModelConfig(**(C1 if args.config == "c1" else MID), eps_assoc=args.eps)
    w = conditioned_weights(cfg)
    S = args.segments
    tokens = cli_tokens(cfg, S * cfg.segment_size - 13, seed=2)
    segs, _ = segment_input(tokens, cfg)
    ids = torch.as_tensor(np.concatenate(segs)).cuda()
    p = prepare_weights(w, args.dtype)
    plan = diagonal_plan(S, cfg.n_layers)
    e = Engine(p, plan.max_members, plan.n_slots)
    st = MemoryState.fresh(cfg)
    st.sync_shadow(p)
    stream = torch.cuda.current_stream().cuda_stream
    d, dm = cfg.d_model, cfg.d_mem
    worst = 0.0
    for step in plan.steps:
        for s, slot in step.enters:
            e.embed(ids[s * cfg.segment_size:(s + 1) * cfg.segment_size], slot, stream)
        e.retrieve(step.slots, step.layers, st, stream)
        e.forward(step.slots, step.layers, stream)
        e.project_kvb(step.slots, step.layers, stream)
        torch.cuda.synchronize()
        before = [(st.A[l].double().cpu().numpy(), st.z[l].double().cpu().numpy()) for l in step.layers]
        kvb = e.kvb[:len(step.layers)].cpu().numpy()
        e.fold(step.slots, step.layers, st, stream)
        torch.cuda.synchronize()
        for g, nd in enumerate(step.nodes):
            l = nd.layer
            A0, z0 = before[g]
            k = kvb[g, :, p.k_off:p.k_off + dm]
            v = kvb[g, :, p.v_off:p.v_off + d]
            b = kvb[g, :, p.b_off]
            A64, z64, zq_m, nrm_m = fold64(A0, z0, k, v, b, cfg.dpfp_nu, p.eps_assoc)
            eA = rel(st.A[l].double().cpu().numpy(), A64)
            ez = rel(st.z[l].double().cpu().numpy(), z64)
            dA = rel(st.A[l].double().cpu().numpy() - A0, A64 - A0)
            worst = max(worst, eA)
            print(json.dumps({"segment": nd.segment, "layer": l, "rel_A": eA, "rel_z": ez, "rel_dA": dA,
                              "zq_margin": zq_m, "nrm_margin": nrm_m}), flush=True)
    print(json.dumps({"worst_rel_A": worst}))


if __name__ == "__main__":
    main()
