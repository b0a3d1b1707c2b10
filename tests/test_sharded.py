"""Layer-sharded pipeline: plan invariants and a world-size-2 gloo run on CPU.

The CPU run drives the product's ``run_stage``/``stage_plan`` with an oracle
backend (test-only) and torch.distributed gloo point-to-point, and must equal
the unsharded oracle diagonal run bitwise (every cell is computed by the same
arithmetic; only the placement and the hand-offs change).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import C1
from paper_2506_05229_b200.config import ModelConfig
from paper_2506_05229_b200.scheduler import diagonal_members
from paper_2506_05229_b200.sharded import TorchP2P, layer_blocks, run_stage, stage_plan, vocab_blocks


@pytest.mark.parametrize("V,P", [(256, 2), (128256, 8), (1000, 3), (300, 4), (50, 1)])
def test_vocab_blocks_partition_and_align(V, P):
    blocks = vocab_blocks(V, P)
    assert len(blocks) == P and blocks[0].start == 0 and blocks[-1].stop == V
    for a, b in zip(blocks, blocks[1:]):
        assert a.stop == b.start
    for b in blocks:
        assert len(b) == 0 or b.start % 64 == 0


@pytest.mark.parametrize("S,L,P", [(8, 16, 2), (128, 16, 8), (3, 5, 4), (1, 4, 4), (10, 7, 3), (5, 2, 1)])
def test_stage_plans_cover_the_wavefront(S, L, P):
    plans = [stage_plan(S, L, r, P) for r in range(P)]
    assert [p.layers for p in plans] == layer_blocks(L, P)
    for i in range(S + L - 1):
        union = [n for p in plans for n in p.steps[i].nodes]
        assert union == diagonal_members(i, S, L)
    for r, p in enumerate(plans):
        for i, st in enumerate(p.steps):
            if st.recv is not None:  # matched by rank r-1's send one step earlier
                assert plans[r - 1].steps[i - 1].send == (st.recv[0], plans[r - 1].steps[i - 1].send[1])
            if st.exits:
                assert r == P - 1
            # every rank joins the vocab-parallel head of the segment leaving layer L-1
            s_exit = i - (L - 1)
            assert st.head == ((s_exit, s_exit % p.n_slots if r == P - 1 else None) if 0 <= s_exit < S else None)
            if st.enter:
                assert r == 0
            # no two in-flight segments share a slot on this rank
            inflight = {n.segment for n in st.nodes}
            slots = [s % p.n_slots for s in inflight]
            assert len(set(slots)) == len(slots)
            for n, slot in zip(st.nodes, st.slots):
                assert slot == n.segment % p.n_slots


class OracleBackend:
    """Test-only backend: oracle cells on CPU tensors (gloo moves them)."""

    def __init__(self, orc, layers, n_slots, tokens, vocab):
        import armt_oracle as O
        self.orc = orc
        self.vocab = vocab
        self.head_in = torch.zeros(orc.cfg.segment_size, orc.cfg.d_model, dtype=torch.float64)
        self.state = O.OracleState.fresh(orc.cfg, np.float64)
        self.slots = [torch.zeros(orc.T, orc.cfg.d_model, dtype=torch.float64) for _ in range(n_slots)]
        self.segs, self.n = O.segment_input(tokens, orc.cfg)
        self.rows = {}

    def slot_tensor(self, slot):
        return self.slots[slot]

    def after_recv(self, slot):
        pass

    def embed(self, s, slot):
        self.slots[slot].copy_(torch.from_numpy(self.orc.embed(self.segs[s])))

    def step(self, slots, layers):
        for slot, l in zip(slots, layers):
            y = self.orc.cell(self.state, l, self.slots[slot].numpy().copy())
            self.slots[slot].copy_(torch.from_numpy(y))

    def head_buffer(self, slot):
        return self.slots[slot][:self.orc.cfg.segment_size] if slot is not None else self.head_in

    def head(self, s, buf):
        self.rows[s] = buf.numpy() @ self.orc.unembedding[:, self.vocab.start:self.vocab.stop]


def _worker(rank, world, port, tokens, out_q):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
    import armt_oracle as O
    from fixtures import conditioned_weights
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = ModelConfig(**C1, eps_assoc=1.0)
    orc = O.Oracle(conditioned_weights(cfg), cfg, np.float64)
    S = len(tokens) // cfg.segment_size
    plan = stage_plan(S, cfg.n_layers, rank, world)
    be = OracleBackend(orc, plan.layers, plan.n_slots, tokens, vocab_blocks(cfg.vocab_size, world)[rank])
    run_stage(plan, be, TorchP2P(dist))
    own = [l for l in plan.layers]
    out_q.put((rank, be.rows, be.state.A[own].copy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_rank_gloo_pipeline_equals_unsharded_oracle():
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))
    import armt_oracle as O
    from fixtures import cli_tokens, conditioned_weights
    cfg = ModelConfig(**C1, eps_assoc=1.0)
    tokens = cli_tokens(cfg, 5 * cfg.segment_size, seed=11)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tokens, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict()
    for _ in range(2):
        r, rows, A = q.get(timeout=300)
        results[r] = (rows, A)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want, wstate, _ = O.Oracle(conditioned_weights(cfg), cfg, np.float64).run_diagonal(tokens)
    # vocab-parallel head: rank r holds the logits of its vocab block for every segment
    got = np.concatenate([np.concatenate([results[r][0][s] for s in range(5)]) for r in range(2)], axis=1)
    assert got.shape == want.shape
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)
    assert np.array_equal(results[0][1], wstate.A[0:1])
    assert np.array_equal(results[1][1], wstate.A[1:2])


class _LogComm:
    """Records the order of communication calls (no data moves)."""

    def __init__(self, log):
        self.log = log

    def isend(self, t, dst):
        self.log.append(("isend", dst, id(t)))
        log, key = self.log, id(t)

        class _W:
            def wait(self_inner):
                log.append(("wait", key))
        return _W()

    def recv(self, t, src):
        self.log.append(("recv", src, id(t)))

    def broadcast(self, t, src):
        self.log.append(("broadcast", src))


class _LogBackend:
    def __init__(self, log, n_slots):
        self.log = log
        self.slots = [torch.zeros(1) for _ in range(n_slots)]

    def slot_tensor(self, slot):
        return self.slots[slot]

    def after_recv(self, slot):
        pass

    def embed(self, s, slot):
        self.log.append(("embed", id(self.slots[slot])))

    def step(self, slots, layers):
        self.log.append(("step", tuple(layers)))

    def head_buffer(self, slot):
        return self.slots[slot] if slot is not None else torch.zeros(1)

    def head(self, s, buf):
        self.log.append(("head", s))


@pytest.mark.parametrize("S,L,P", [(8, 16, 4), (20, 16, 8), (5, 6, 3), (3, 4, 2)])
def test_stage_ordering_sends_before_collective_and_no_slot_reuse_in_flight(S, L, P):
    """Every rank posts a step's cells and its send BEFORE the deferred head
    broadcast of that step (the head is off the path between a rank's cells and
    the send its successor waits for), and no slot with a send in flight is
    rewritten (received into or embedded) before that send was waited on."""
    for r in range(P):
        plan = stage_plan(S, L, r, P)
        log = []
        run_stage(plan, _LogBackend(log, plan.n_slots), _LogComm(log))
        in_flight = set()
        for ev in log:
            if ev[0] == "isend":
                assert ev[2] not in in_flight
                in_flight.add(ev[2])
            elif ev[0] == "wait":
                in_flight.discard(ev[1])
            elif ev[0] in ("recv", "embed"):
                buf = ev[2] if ev[0] == "recv" else ev[1]
                assert buf not in in_flight, (r, ev)
        heads = [k for k, ev in enumerate(log) if ev[0] == "head"]
        assert [log[k][1] for k in heads] == list(range(S))
        if P > 1:
            assert sum(1 for ev in log if ev[0] == "broadcast") == S
        idx_step = [k for k, ev in enumerate(log) if ev[0] == "step"]
        idx_send = [k for k, ev in enumerate(log) if ev[0] == "isend"]
        cell_steps = [i for i, st in enumerate(plan.steps) if st.nodes]
        for s, k in enumerate(heads):
            i_head = s + L   # segment s leaves layer L-1 at step s+L-1; its head runs after step s+L's work
            done = {i for i, kk in zip(cell_steps, idx_step) if kk < k}
            assert done == {i for i in cell_steps if i <= i_head}
            sends = sum(1 for kk in idx_send if kk < k)
            assert sends == sum(1 for st in plan.steps[:i_head + 1] if st.send is not None)
