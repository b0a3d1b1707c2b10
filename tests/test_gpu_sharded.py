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


def test_sharded_session_single_rank_matches_session():
    """ShardedSession (per-step CUDA graphs, vocab-parallel head code path) at
    world size 1 reproduces the single-GPU Session bitwise: logits and the
    fused-NLL scoring output."""
    from paper_2506_05229_b200.executors import Session
    from paper_2506_05229_b200.sharded import ShardedSession
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    w = conditioned_weights(cfg)
    n = 5 * cfg.segment_size - 3
    tokens = torch.as_tensor(cli_tokens(cfg, n, seed=5)).cuda()
    ref = Session(prepare_weights(w, "bf16"), n)
    want = ref.forward(tokens).clone()
    sh = ShardedSession(w, cfg, n, rank=0, world=1)
    sh._load_ids(tokens)
    sh.warm()
    got = sh.forward()
    assert torch.equal(got, want)
    ref_s = Session(prepare_weights(w, "bf16"), n, scoring=True)
    want_nll = ref_s.nll(tokens).clone()
    sh_s = ShardedSession(w, cfg, n, rank=0, world=1, scoring=True)
    sh_s._load_ids(tokens)
    sh_s.warm()
    got_nll = sh_s.nll()
    assert torch.allclose(got_nll, want_nll, rtol=1e-5, atol=1e-5)


def test_sharded_capture_keeps_one_graph_per_launch_sequence():
    """Steps with the same (slots, layers) repeat as the slots cycle; the capture
    pass keeps ONE graph per distinct launch sequence and every kept graph is
    replayed (a re-captured duplicate used to replace the first graph, orphaning
    anything recorded in it, e.g. the bench's in-graph roofline probe events)."""
    from paper_2506_05229_b200.sharded import ShardedSession
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    w = conditioned_weights(cfg)
    n = 12 * cfg.segment_size
    tokens = torch.as_tensor(cli_tokens(cfg, n, seed=9)).cuda()
    sh = ShardedSession(w, cfg, n, rank=0, world=1)
    sh._load_ids(tokens)
    sh.warm_eager()
    eager = sh.forward().clone()
    sh.capture()
    graphs = sh.backend.graphs
    step_keys = [k for k in graphs if k[0] == "step"]
    assert len(step_keys) < sum(1 for st in sh.plan.steps if st.nodes)   # repeats exist at 12 segments
    used = set()

    class Counting:
        def __init__(self, key, g):
            self.key, self.g = key, g

        def replay(self):
            used.add(self.key)
            self.g.replay()

    for k in list(graphs):
        graphs[k] = Counting(k, graphs[k])
    got = sh.forward()
    assert torch.equal(got, eager)
    assert used == set(graphs)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_vocab_parallel_nll_combine_matches_full_vocab(P):
    """Per-rank vocab blocks -> fused LSE partials -> per-row (max, sum) ->
    cross-rank finalize equals the NLL of the full-vocab logits (the math of
    ShardedSession.nll with the all-gather done in one process)."""
    from paper_2506_05229_b200 import _lib
    from paper_2506_05229_b200.sharded import vocab_blocks
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    w = conditioned_weights(cfg)
    p = prepare_weights(w, "bf16")
    eng = Engine(p, 1, 1)
    seg, d, V = cfg.segment_size, cfg.d_model, cfg.vocab_size
    torch.manual_seed(0)
    x = torch.randn(seg, d, device="cuda").bfloat16()
    n = seg + 1
    ids = torch.randint(0, V, (n + seg,), device="cuda")
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    full = torch.empty(seg, V, dtype=torch.float32, device="cuda")
    eng.unembed_block(x.data_ptr(), d, 0, V, 0, st, out=full)
    want = torch.empty(seg, device="cuda")
    _lib.check(lib.armt_logits_nll(full.data_ptr(), _lib.F32, V, ids[1:].data_ptr(), want.data_ptr(), seg, V, st), "nll")
    ms = torch.empty(seg, P, 2, device="cuda")
    tgt_sum = torch.zeros(seg, device="cuda")
    for r, blk in enumerate(vocab_blocks(V, P)):
        if not len(blk):
            ms[:, r, 0] = float("-inf"); ms[:, r, 1] = 0
            continue
        tiles = -(-len(blk) // 256)
        part = torch.empty(seg, tiles, 2, device="cuda")
        tgt = torch.zeros(seg, device="cuda")
        loc = ids - blk.start
        eng.unembed_block(x.data_ptr(), d, blk.start, blk.stop, 0, st, lse=(part, tgt, loc, n))
        row = torch.empty(seg, 2, device="cuda")
        _lib.check(lib.armt_lse_reduce(part.data_ptr(), tiles, tiles, row.data_ptr(), seg, st), "reduce")
        ms[:, r] = row
        tgt_sum += tgt
    got = torch.empty(seg, device="cuda")
    _lib.check(lib.armt_lse_finalize(ms.data_ptr(), P, P, tgt_sum.data_ptr(), ids[1:].data_ptr(), got.data_ptr(),
                                     seg, st), "finalize")
    assert torch.allclose(got, want, rtol=1e-4, atol=1e-4), (got - want).abs().max()


def _two_rank_worker(rank, world, port, out_q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    from conftest import MID as _MID
    from fixtures import cli_tokens as _tok, conditioned_weights as _cw
    from paper_2506_05229_b200.config import ModelConfig as _MC
    from paper_2506_05229_b200.sharded import ShardedSession
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _MC(**_MID, eps_assoc=10.0)
    w = _cw(cfg)
    n = 5 * cfg.segment_size - 3
    tokens = torch.as_tensor(_tok(cfg, n, seed=5)).cuda()
    sh = ShardedSession(w, cfg, n, rank=rank, world=world)
    sh._load_ids(tokens)
    sh.warm()
    logits = sh.forward().float().cpu()
    sc = ShardedSession(w, cfg, n, rank=rank, world=world, scoring=True)
    sc._load_ids(tokens)
    sc.warm()
    nll = sc.nll().cpu()
    out_q.put((rank, sh.vocab, logits, nll))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_pipeline_on_one_gpu_matches_single_session():
    """World-size-2 layer-sharded run (two processes sharing this GPU, gloo
    with host-staged hand-offs): the vocab-parallel logit blocks reassemble the
    single-GPU logits bitwise and the all-gathered NLL matches."""
    import socket
    import torch.multiprocessing as mp
    from paper_2506_05229_b200.executors import Session
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, vocab, logits, nll = q.get(timeout=600)
        res[r] = (vocab, logits, nll)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    w = conditioned_weights(cfg)
    n = 5 * cfg.segment_size - 3
    tokens = torch.as_tensor(cli_tokens(cfg, n, seed=5)).cuda()
    want = Session(prepare_weights(w, "bf16"), n).forward(tokens).float().cpu()
    got = torch.cat([res[0][1], res[1][1]], dim=1)
    assert res[0][0].stop == res[1][0].start and got.shape == want.shape
    assert torch.equal(got, want)
    want_nll = Session(prepare_weights(w, "bf16"), n, scoring=True).nll(tokens).cpu()
    for r in range(2):
        assert torch.allclose(res[r][2], want_nll, rtol=1e-5, atol=1e-5)
