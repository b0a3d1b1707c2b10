"""Per-segment-count error and liveness table for the C2 bench fixture (GPU).

    python scripts/c2_horizon_table.py [--segments 128] [--cols 16384] [--modes f32,bf16,...]

The bench fixture: C2 (L16 d2048 H32 ff8192 seg1024 M128 d_mem64 V128256),
the reference initialiser (seed 0), w_v_mem x 1/32, eps_assoc 100, weights on
the bf16 grid (so every mode sees identical weights), cli token convention.

Every mode runs the diagonal schedule eagerly through this package's engine
(the same kernels the bench graph replays) with a per-segment LM head; the
first ``--cols`` vocabulary columns of each segment's logits are compared with
the device f32 parity run. Because the forward is causal over segments, the
error on segment s is the error "after s+1 segments": one run gives the whole
horizon table.

Modes
  f32           parity mode (fp32 SIMT GEMMs, in-order fp32 fold): the reference
  bf16          production path (fused norms, tcgen05 GEMMs, tensor-core fold)
  bf16_fold32   bf16, but the memory update (k/v/beta projection + fold) in fp32
  bf16_mem32    bf16 backbone, memory read AND update in fp32
  bf16_kvb32    bf16, k/v/beta projection in fp32 from the fp32 stream, tensor-core fold
  bf16_tcfold32 bf16, bf16 k/v/beta projection, fp32 in-order fold (isolates the fold)
  f32_inert     f32 with W_k = 0: the memory never stores anything (liveness)
  bf16_inert    bf16 with W_k = 0

Also prints the fraction of retrieval rows whose |phi.z| <= eps_assoc (guarded
to zero) per segment, from the f32 run. One JSON line per result.
"""

from __future__ import annotations

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

from paper_2506_05229_b200 import ModelConfig, init_weights, round_to_bf16  # noqa: E402
from paper_2506_05229_b200.engine import Engine, MemoryState, prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import diagonal_plan  # noqa: E402

C2 = dict(n_layers=16, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024, num_mem_tokens=128,
          d_mem=64, vocab_size=128256)


def emit(**kw):
    print(json.dumps(kw), flush=True)


def run_mode(mode, w_b, w_f, cfg, ids, S, cols, guard=None):
    """Eager diagonal run; returns (S*seg, cols) f32 logits slice on device and final A."""
    inert = mode.endswith("_inert")
    base = mode.replace("_inert", "")
    dev = torch.device("cuda")
    plan = diagonal_plan(S, cfg.n_layers)
    G = plan.max_members
    seg = cfg.segment_size
    need_b = base != "f32"
    need_f = base != "bf16"
    pb = prepare_weights(w_b if not inert else replace(w_b, w_k_mem=np.zeros_like(w_b.w_k_mem)), "bf16") \
        if need_b else None
    pf = prepare_weights(w_f if not inert else replace(w_f, w_k_mem=np.zeros_like(w_f.w_k_mem)), "f32") \
        if need_f else None
    fused = base in ("bf16", "bf16_fold32", "bf16_kvb32", "bf16_tcfold32")
    eb = Engine(pb, G, plan.n_slots, fused_norm=fused) if need_b else None
    ef = Engine(pf, G, plan.n_slots, slots_from=eb) if need_f else None
    e_ret = ef if base in ("f32", "bf16_mem32") else eb
    e_fwd = ef if base == "f32" else eb
    e_upd = ef if base in ("f32", "bf16_fold32", "bf16_mem32") else eb
    state = MemoryState.fresh(cfg)
    if need_b:
        state.sync_shadow(pb)
    stream = torch.cuda.current_stream().cuda_stream
    out = torch.empty(S * seg, cols, device=dev)
    lm = torch.empty(seg, cfg.vocab_size, dtype=torch.bfloat16 if e_fwd is eb else torch.float32, device=dev)
    eps = (pf or pb).eps_assoc
    t0 = time.time()
    for st in plan.steps:
        for s, slot in st.enters:
            e_fwd.embed(ids[s * seg:(s + 1) * seg], slot, stream)
        e_ret.retrieve(st.slots, st.layers, state, stream)
        if guard is not None:
            den = e_ret.den[:len(st.layers)].abs() <= eps
            for g, nd in enumerate(st.nodes):
                guard.setdefault(nd.segment, []).append(float(den[g].float().mean()))
        e_fwd.forward(st.slots, st.layers, stream)
        for s, slot in st.exits:
            e_fwd.unembed(slot, lm, 0, stream)
            out[s * seg:(s + 1) * seg] = lm[:, :cols].float()
        if base == "bf16_kvb32":      # fp32 k/v/beta projection (from the fp32 stream), tensor-core fold
            ef.project_kvb(st.slots, st.layers, stream)
            eb.kvb[:len(st.layers)].copy_(ef.kvb[:len(st.layers)])
            eb.fold(st.slots, st.layers, state, stream)
        elif base == "bf16_tcfold32":  # bf16 projection (from the bf16 stream copy), fp32 in-order fold
            eb.project_kvb(st.slots, st.layers, stream)
            ef.kvb[:len(st.layers)].copy_(eb.kvb[:len(st.layers)])
            ef.fold(st.slots, st.layers, state, stream)
            state.sync_shadow(pb)
        else:
            e_upd.update(st.slots, st.layers, state, stream)
            if e_upd is ef and need_b and e_ret is eb:
                state.sync_shadow(pb)   # the bf16 retrieval reads the split operand; refresh it from fp32 A, z
    torch.cuda.synchronize()
    dt = time.time() - t0
    A = state.A.clone()
    del eb, ef, pb, pf, lm, state
    torch.cuda.empty_cache()
    return out, A, dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--segments", type=int, default=128)
    ap.add_argument("--cols", type=int, default=16384)
    ap.add_argument("--eps", type=float, default=100.0)
    ap.add_argument("--modes", default="f32,bf16,bf16_fold32,bf16_mem32,f32_inert")
    args = ap.parse_args()
    cfg = ModelConfig(**C2, eps_assoc=args.eps, seed=0)
    t = time.time()
    w = init_weights(cfg, dtype=np.float32)
    w = replace(w, w_v_mem=w.w_v_mem * np.float32(1 / 32)).map_arrays(round_to_bf16)
    emit(event="init", seconds=time.time() - t, eps_assoc=args.eps)
    S = args.segments
    n = S * cfg.segment_size
    tokens = np.random.default_rng([0, n]).integers(0, cfg.vocab_size, n, dtype=np.int64)
    ids = torch.as_tensor(tokens).cuda()
    seg = cfg.segment_size
    ref = None
    refA = None
    guard: dict = {}
    per_mode = {}
    for mode in args.modes.split(","):
        logits, A, dt = run_mode(mode, w, w, cfg, ids, S, args.cols, guard if mode == "f32" else None)
        finite = [bool(torch.isfinite(logits[s * seg:(s + 1) * seg]).all()) for s in range(S)]
        emit(event="mode_done", mode=mode, seconds=dt, all_finite=all(finite),
             first_nonfinite=(finite.index(False) if not all(finite) else None))
        if mode == "f32":
            ref, refA = logits, A
            continue
        errs = []
        for s in range(S):
            a, b = logits[s * seg:(s + 1) * seg].double(), ref[s * seg:(s + 1) * seg].double()
            errs.append(float((a - b).norm() / b.norm()))
        per_mode[mode] = errs
        emit(event="per_segment_rel_err_vs_f32", mode=mode, errors=errs,
             final_A_rel_err=float((A.double() - refA.double()).norm() / refA.double().norm()))
        del logits
        torch.cuda.empty_cache()
    if guard:
        emit(event="guarded_row_fraction_f32", per_segment=[float(np.mean(guard[s])) for s in range(S)])
    table = {}
    for k in (1, 2, 4, 8, 16, 32, 64, 128):
        if k <= S:
            table[k] = {m: per_mode[m][k - 1] for m in per_mode}
            table[k]["guarded"] = float(np.mean(guard[k - 1])) if guard else None
    emit(event="table", after_segments=table)


if __name__ == "__main__":
    main()
