"""Spread of the C1 bf16 end-to-end error (logits / A / z vs the f64 oracle) over token
seeds, to tell a systematic fold change from chaotic amplification of rounding noise.
A/B the fold with ARMT_FOLD_V1=1."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import armt_oracle as O  # noqa: E402
from conftest import C1  # noqa: E402
from fixtures import cli_tokens, conditioned_weights  # noqa: E402
from paper_2506_05229_b200 import ModelConfig  # noqa: E402
from paper_2506_05229_b200.engine import MemoryState, prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import relative_error as rel, run_diagonal  # noqa: E402

tag = "v1" if os.environ.get("ARMT_FOLD_V1") == "1" else "v2"
cfg = ModelConfig(**C1, eps_assoc=1.0)
w = conditioned_weights(cfg)
prep = prepare_weights(w, "bf16")
orc = O.Oracle(w, cfg, np.float64)
res = []
for seed in range(12):
    toks = cli_tokens(cfg, 8 * cfg.segment_size, seed=seed)
    want, ost, _ = orc.run_diagonal(toks)
    st = MemoryState.fresh(cfg)
    lg, _ = run_diagonal(prep, cfg, toks, state=st, graph=False)
    A, z, _ = st.to_numpy()
    res.append((rel(lg, want), rel(A, ost.A), rel(z, ost.z)))
    print(tag, seed, "logits %.3e A %.3e z %.3e" % res[-1], flush=True)
r = np.array(res)
print(tag, "median", np.median(r, 0), "max", r.max(0))
