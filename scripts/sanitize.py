"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): one eager
diagonal + sequential forward of a small config through every production kernel
path, bf16 and f32. Usage: python scripts/sanitize.py {c1,mid,c2w}"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import C1, MID  # noqa: E402
from fixtures import cli_tokens, conditioned_weights  # noqa: E402
from paper_2506_05229_b200 import ModelConfig  # noqa: E402
from paper_2506_05229_b200.engine import MemoryState, prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import Session, run_diagonal, run_sequential  # noqa: E402

CFGS = {
    "c1": (C1, 1.0, 8),     # d_head 32: mma.sync attention
    "mid": (MID, 10.0, 6),  # d_head 64: tcgen05 ping-pong attention
    # C2 layer shapes (2 layers): CTA pairs, multicast clusters, concurrent remainder, fused DPFP
    "c2w": (dict(n_layers=2, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024, num_mem_tokens=128,
                 d_mem=64, vocab_size=4096), 100.0, 2),
}

name = sys.argv[1]
model, eps, S = CFGS[name]
cfg = ModelConfig(**model, eps_assoc=eps, seed=0)
w = conditioned_weights(cfg)
tokens = cli_tokens(cfg, S * cfg.segment_size - 5)
for dtype in ("bf16", "f32"):
    prep = prepare_weights(w, dtype, device="cuda:0")
    st = MemoryState.fresh(cfg, "cuda:0")
    a, _ = run_diagonal(prep, cfg, tokens, dtype=dtype, state=st, graph=False)
    b, _ = run_sequential(prep, cfg, tokens, dtype=dtype, graph=False)
    assert np.array_equal(a, b), f"{name} {dtype}: schedules disagree"
    assert np.isfinite(a).all()
    print(f"{name} {dtype}: ok", flush=True)
prep = prepare_weights(w, "bf16", device="cuda:0")
ses = Session(prep, len(tokens), graph=False, scoring=True)
nll = ses.nll(torch.as_tensor(tokens))
torch.cuda.synchronize()
print(f"{name} scoring: ok mean nll {float(nll.mean()):.4f}", flush=True)
