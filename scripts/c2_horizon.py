"""Sweep C2 fixture conditioning over the full 128-segment horizon on the device.

For each (eps_assoc, damp, qk_scale): first non-finite segment and NLL drift
in f32 (parity mode, ~1e-5 of the oracle at 2 segments) and bf16, plus the
bf16-vs-f32 relative logits error on the last segments.
"""

import argparse
import json
import os
import sys
from dataclasses import replace

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2506_05229_b200 import ModelConfig, init_weights, round_to_bf16  # noqa: E402
from paper_2506_05229_b200.engine import prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import Session, relative_error  # noqa: E402

C2 = dict(n_layers=16, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024, num_mem_tokens=128,
          d_mem=64, vocab_size=128256)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="10,0.03125,1;100,0.03125,1;10,0.03125,0.5;1000,0.03125,1")
    ap.add_argument("--horizon", type=int, default=128)
    args = ap.parse_args()
    base = init_weights(ModelConfig(**C2, seed=0), dtype=np.float32)
    n = args.horizon * 1024
    tokens = torch.as_tensor(np.random.default_rng([0, n]).integers(0, 128256, n, dtype=np.int64)).cuda()
    for item in args.grid.split(";"):
        eps, damp, qk = (float(v) for v in item.split(","))
        cfg = ModelConfig(**C2, eps_assoc=eps, seed=0)
        w = replace(base, config=cfg, w_v_mem=base.w_v_mem * np.float32(damp),
                    w_k_mem=base.w_k_mem * np.float32(qk), w_q_assoc=base.w_q_assoc * np.float32(qk))
        w = w.map_arrays(round_to_bf16)
        out = {"eps": eps, "damp": damp, "qk_scale": qk}
        tail = {}
        for dt in ("f32", "bf16"):
            prep = prepare_weights(w, dt)
            sess = Session(prep, n, graph=False)
            nll = sess.nll(tokens).float().cpu().numpy()
            per = nll[:n - 1].reshape(-1)[: (args.horizon * 1024 - 1)]
            seg = [float(np.mean(per[s * 1024:(s + 1) * 1024 - 1])) for s in range(args.horizon)]
            bad = [s for s, v in enumerate(seg) if not np.isfinite(v)]
            out[f"{dt}_first_nonfinite"] = bad[0] if bad else None
            out[f"{dt}_nll"] = [round(v, 3) for v in (seg[0], seg[len(seg) // 2], seg[-1])]
            out[f"{dt}_A_norm"] = float(sess.state.A.norm())
            tail[dt] = sess.runner.logits[(args.horizon - 2) * 1024:args.horizon * 1024].float().cpu()
            del sess, prep
            torch.cuda.empty_cache()
        out["bf16_vs_f32_last2seg"] = relative_error(tail["bf16"], tail["f32"])
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
