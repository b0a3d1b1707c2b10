"""Layer-sharded device path on ONE GPU (``-m gpu``).

All P stages run in one process, each with its own layer block of prepared
weights, its own partial memory state and its own Engine (exactly what each
rank holds); the P2P hand-off is a device copy through a mailbox. The result
must equal the unsharded device diagonal run bitwise.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from conftest import C1, MID  # noqa: E402
from fixtures import cli_tokens, conditioned_weights  # noqa: E402
from paper_2506_05229_b200.config import ModelConfig  # noqa: E402
from paper_2506_05229_b200.engine import Engine, MemoryState, prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import run_diagonal  # noqa: E402
from paper_2506_05229_b200.sharded import DeviceBackend, stage_plan  # noqa: E402


def run_local_pipeline(w, cfg, tokens, world):
    S = -(-len(tokens) // cfg.segment_size)
    ids = torch.zeros(S * cfg.segment_size, dtype=torch.int64, device="cuda")
    ids[:len(tokens)] = torch.as_tensor(tokens)
    logits = torch.empty(S * cfg.segment_size, cfg.vocab_size, dtype=torch.bfloat16, device="cuda")
    stream = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    plans, backs, states = [], [], []
    for r in range(world):
        plan = stage_plan(S, cfg.n_layers, r, world)
        p = prepare_weights(w, "bf16", layers=plan.layers)
        st = MemoryState.fresh(cfg, n_layers=len(plan.layers))
        st.sync_shadow(p)
        eng = Engine(p, plan.max_members, plan.n_slots)
        plans.append(plan)
        states.append(st)
        backs.append(DeviceBackend(eng, ids, logits, st, cfg.segment_size, stream))
    mailbox = {}
    for i in range(S + cfg.n_layers - 1):
        for r in range(world):
            st, be = plans[r].steps[i], backs[r]
            if st.recv is not None:
                s, slot = st.recv
                be.slot_tensor(slot).copy_(mailbox.pop((r, s)))
                be.after_recv(slot)
            if st.enter is not None:
                be.embed(*st.enter)
            if st.nodes:
                be.step(st.slots, st.layers)
            if st.send is not None:
                s, slot = st.send
                mailbox[(r + 1, s)] = be.slot_tensor(slot).clone()
            for s, slot in st.exits:
                be.unembed(s, slot)
    torch.cuda.synchronize()
    A = torch.cat([s.A for s in states]).cpu().numpy()
    return logits[:len(tokens)].float().cpu().numpy(), A


@pytest.mark.parametrize("conf,eps,world", [(C1, 1.0, 2), (MID, 10.0, 2), (MID, 10.0, 4), (MID, 10.0, 3)])
def test_local_pipeline_equals_unsharded(conf, eps, world):
    cfg = ModelConfig(**conf, eps_assoc=eps)
    w = conditioned_weights(cfg)
    tokens = cli_tokens(cfg, 5 * cfg.segment_size - 3, seed=21)
    got, A = run_local_pipeline(w, cfg, tokens, world)
    st = MemoryState.fresh(cfg)
    want, _ = run_diagonal(prepare_weights(w, "bf16"), cfg, tokens, state=st)
    assert np.array_equal(got, want)
    assert np.array_equal(A, st.A.cpu().numpy())
