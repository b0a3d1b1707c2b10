"""C1 / MID bf16 errors vs the reference goldens / f64 oracle (A/B the fold with ARMT_FOLD_V1=1)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import armt_oracle as O  # noqa: E402
from conftest import C1, MID, golden  # noqa: E402
from fixtures import cli_tokens, conditioned_weights  # noqa: E402
from paper_2506_05229_b200 import ModelConfig  # noqa: E402
from paper_2506_05229_b200.engine import MemoryState, prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import relative_error as rel, run_diagonal  # noqa: E402

tag = "v1" if os.environ.get("ARMT_FOLD_V1") == "1" else "v2"
cfg = ModelConfig(**C1, eps_assoc=1.0)
w = conditioned_weights(cfg)
g = golden("c1_cond")
st = MemoryState.fresh(cfg)
lg, _ = run_diagonal(prepare_weights(w, "bf16"), cfg, g["tokens"], state=st, graph=False)
A, z, _ = st.to_numpy()
print(tag, "C1 logits %.3e A %.3e z %.3e" % (rel(lg, g["logits_f64"]), rel(A, g["A_f64"]), rel(z, g["z_f64"])))
cfg = ModelConfig(**MID, eps_assoc=10.0)
w = conditioned_weights(cfg)
toks = cli_tokens(cfg, 6 * cfg.segment_size - 13)
want, ost, _ = O.Oracle(w, cfg, np.float64).run_diagonal(toks)
st = MemoryState.fresh(cfg)
lg, _ = run_diagonal(prepare_weights(w, "bf16"), cfg, toks, state=st, graph=False)
A, z, _ = st.to_numpy()
print(tag, "MID logits %.3e A %.3e z %.3e" % (rel(lg, want), rel(A, ost.A), rel(z, ost.z)))
