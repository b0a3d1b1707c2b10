"""C2 (LLaMA-1B-shaped) numerics on the device: parity with the oracle over
the first segments, and finiteness/drift over a long horizon.

    python scripts/c2_check.py [--eps 10] [--segments 2] [--horizon 128]

Prints one JSON line per measurement (used for DESIGN.md's parity table).
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import armt_oracle as O  # noqa: E402
from paper_2506_05229_b200 import ModelConfig, init_weights, round_to_bf16  # noqa: E402
from paper_2506_05229_b200.engine import MemoryState, prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import Session, relative_error, run_diagonal  # noqa: E402
from dataclasses import replace  # noqa: E402

C2 = dict(n_layers=16, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024, num_mem_tokens=128,
          d_mem=64, vocab_size=128256)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eps", type=float, default=10.0)
    ap.add_argument("--damp", type=float, default=1 / 32)
    ap.add_argument("--segments", type=int, default=2)
    ap.add_argument("--horizon", type=int, default=128)
    ap.add_argument("--qk-scale", type=float, default=1.0, help="scale W_k_mem and W_q_assoc")
    args = ap.parse_args()
    cfg = ModelConfig(**C2, eps_assoc=args.eps, seed=0)
    t = time.time()
    w = init_weights(cfg, dtype=np.float32)
    w = replace(w, w_v_mem=w.w_v_mem * np.float32(args.damp),
                w_k_mem=w.w_k_mem * np.float32(args.qk_scale), w_q_assoc=w.w_q_assoc * np.float32(args.qk_scale))
    w = w.map_arrays(round_to_bf16)
    print(json.dumps({"init_s": time.time() - t}), flush=True)
    n = args.segments * cfg.segment_size
    tokens = np.random.default_rng([0, n]).integers(0, cfg.vocab_size, n, dtype=np.int64)

    # device runs
    res = {}
    for dt in ("bf16", "f32"):
        prep = prepare_weights(w, dt)
        st = MemoryState.fresh(cfg)
        logits, _ = run_diagonal(prep, cfg, tokens, dtype=dt, state=st)
        res[dt] = (logits, st.A.cpu().numpy(), st.z.cpu().numpy())
        del prep
        torch.cuda.empty_cache()
    # oracle (f32 numpy, host cores)
    t = time.time()
    orc = O.Oracle(w, cfg, np.float32)
    ol, ost, _ = orc.run_sequential(tokens)
    t_or = time.time() - t
    # memory liveness: same run with the memory read disabled (inert keys)
    inert = replace(w, w_k_mem=np.zeros_like(w.w_k_mem))
    il, _, _ = O.Oracle(inert, cfg, np.float32).run_sequential(tokens)
    for dt in ("bf16", "f32"):
        lg, A, z = res[dt]
        print(json.dumps({"check": "c2_parity_vs_oracle_f32", "dtype": dt, "segments": args.segments,
                          "eps": args.eps, "rel_logits": relative_error(lg, ol), "rel_A": relative_error(A, ost.A),
                          "rel_z": relative_error(z, ost.z), "finite": bool(np.isfinite(lg).all()),
                          "oracle_s": t_or}), flush=True)
    print(json.dumps({"check": "c2_memory_liveness", "rel_logits_vs_inert": relative_error(ol, il)}), flush=True)
    del res

    # long horizon: per-segment finiteness and NLL on the bf16 session
    n = args.horizon * cfg.segment_size
    tokens = np.random.default_rng([0, n]).integers(0, cfg.vocab_size, n, dtype=np.int64)
    prep = prepare_weights(w, "bf16")
    sess = Session(prep, n)
    nll = sess.nll(torch.as_tensor(tokens).cuda()).float().cpu().numpy()
    seg = cfg.segment_size
    per_seg = [float(np.mean(nll[s * seg:(s + 1) * seg - 1])) for s in range(args.horizon)]
    bad = [s for s, v in enumerate(per_seg) if not np.isfinite(v)]
    Anorm = sess.state.A.float().norm().item()
    print(json.dumps({"check": "c2_horizon", "segments": args.horizon, "first_nonfinite_segment": bad[0] if bad else None,
                      "nll_first": per_seg[:4], "nll_last": per_seg[-4:], "A_norm": Anorm}), flush=True)


if __name__ == "__main__":
    main()
