"""Full-depth C2 (16 layers, d 2048, V 4096, 3 segments): per-layer memory-state
error of each precision mode against the f32 oracle (GPU + host oracle).

    python scripts/c2_depth_modes.py [--modes f32,bf16,bf16_fold32,bf16_mem32]

Same fixture as tests/test_gpu_parity.py::c2_full_depth. Modes as in
scripts/c2_horizon_table.py. One JSON line per mode: logits / A / z relative
errors overall and per layer.
"""

from __future__ import annotations

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
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import armt_oracle as O  # noqa: E402
from fixtures import cli_tokens, conditioned_weights  # noqa: E402
from paper_2506_05229_b200 import ModelConfig  # noqa: E402
from paper_2506_05229_b200.executors import relative_error, segment_input  # noqa: E402
import c2_horizon_table as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="f32,bf16,bf16_fold32,bf16_mem32")
    ap.add_argument("--segments", type=int, default=3)
    args = ap.parse_args()
    cfg = ModelConfig(n_layers=16, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024, num_mem_tokens=128,
                      d_mem=64, vocab_size=4096, eps_assoc=100.0, seed=0)
    w = conditioned_weights(cfg)
    S = args.segments
    tokens = cli_tokens(cfg, S * cfg.segment_size - 13, seed=2)
    t = time.time()
    want, ostate, _ = O.Oracle(w, cfg, np.float32).run_diagonal(tokens)
    print(json.dumps({"event": "oracle", "seconds": time.time() - t}), flush=True)
    segs, n = segment_input(tokens, cfg)
    ids = torch.as_tensor(np.concatenate(segs)).cuda()
    for mode in args.modes.split(","):
        logits, A, _ = H.run_mode(mode, w, w, cfg, ids, S, cfg.vocab_size)
        lg = logits[:n].cpu().numpy()
        A = A.cpu().numpy()
        print(json.dumps({
            "mode": mode, "rel_logits": relative_error(lg, want),
            "rel_logits_per_segment": [relative_error(lg[s * 1024:(s + 1) * 1024], want[s * 1024:(s + 1) * 1024])
                                       for s in range(S)],
            "rel_A": relative_error(A, ostate.A),
            "rel_A_per_layer": [relative_error(A[l], ostate.A[l]) for l in range(cfg.n_layers)],
        }), flush=True)


if __name__ == "__main__":
    main()
