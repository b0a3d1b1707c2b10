"""Layer-sharded (pipeline-over-the-wavefront) execution on 1..N GPUs.

SURVEY §8(e): the diagonal wavefront shards naturally by layer. Rank r owns
the contiguous layer block [lo_r, hi_r) — its weights and its fp32 memory
state (A, z never move). At global step i it runs the cells {(i-l, l) :
l in [lo_r, hi_r)} as one grouped step. The only cross-rank edge is
(s, lo_r - 1) -> (s, lo_r): after step i-1 rank r-1 sends the activation of
segment s = i - lo_r (its last layer's output, T x d fp32) and rank r receives
it before step i. Rank 0 embeds.

The LM head is vocab-parallel: when segment s clears layer
L-1 at step i, the last rank broadcasts its token rows (seg x d) at the start
of step i+1 (after that step's receive, so every rank's point-to-point
traffic of step i is posted before the collective: no cross-rank ordering
deadlock), and every rank computes the logits of its contiguous vocab block
(``vocab_blocks``). This spreads the 17% LM-head load over all ranks instead
of stalling the pipeline on the last one, and shards the logits / NLL
partials. Scoring sessions combine per-rank (max, sum-exp) row partials with
one all-gather at the end.

``StagePlan`` is the per-rank integer bookkeeping (pure host logic, tested on
CPU with world size 2 over gloo); ``run_stage`` drives any backend exposing
``slot_tensor / after_recv / embed / step / unembed`` — the CUDA ``Engine``
here, an oracle backend in tests/test_sharded.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InputError
from .scheduler import Node, diagonal_members


def vocab_blocks(vocab: int, world: int, align: int = 64) -> list[range]:
    """Contiguous near-even vocab blocks, one per rank, starting on ``align``
    multiples (each rank's NLL partial tiles are local to its block)."""
    per = -(-vocab // world)
    per = -(-per // align) * align
    return [range(min(r * per, vocab), min((r + 1) * per, vocab)) for r in range(world)]


def layer_blocks(n_layers: int, world: int) -> list[range]:
    """Contiguous near-even partition of [0, L) into ``world`` blocks."""
    if world < 1 or world > n_layers:
        raise InputError(f"cannot shard {n_layers} layers over {world} ranks")
    base, rem = divmod(n_layers, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < rem else 0)
        out.append(range(lo, hi))
        lo = hi
    return out


@dataclass
class StageStep:
    nodes: list[Node]            # this rank's cells, ascending layer (reference order)
    slots: list[int]
    layers: list[int]
    recv: tuple[int, int] | None   # (segment, slot) received from rank-1 before the step
    enter: tuple[int, int] | None  # (segment, slot) embedded before the step (rank 0)
    send: tuple[int, int] | None   # (segment, slot) sent to rank+1 after the step
    exits: list[tuple[int, int]]   # (segment, slot) leaving layer L-1 at this step (last rank)
    head: tuple[int, int | None] | None = None  # (segment, last-rank slot or None): every rank


@dataclass
class StagePlan:
    rank: int
    world: int
    n_segments: int
    n_layers: int
    layers: range
    n_slots: int
    steps: list[StageStep]

    @property
    def max_members(self) -> int:
        return max([len(s.nodes) for s in self.steps] + [1])


def stage_plan(n_segments: int, n_layers: int, rank: int, world: int) -> StagePlan:
    S, L = n_segments, n_layers
    blk = layer_blocks(L, world)[rank]
    lo, hi = blk.start, blk.stop
    last = hi == L
    # one spare slot: the exiting segment's rows stay intact until its deferred
    # LM-head broadcast at the start of the next step (after that step's receive)
    n_slots = max(1, min(S, hi - lo + 1))
    steps = []
    for i in range(S + L - 1):
        nodes = [n for n in diagonal_members(i, S, L) if lo <= n.layer < hi]
        slot = lambda s: s % n_slots  # noqa: E731
        s_in = i - lo
        recv = (s_in, slot(s_in)) if lo > 0 and 0 <= s_in < S else None
        enter = (i, slot(i)) if lo == 0 and i < S else None
        s_out = i - (hi - 1)
        send = (s_out, slot(s_out)) if hi < L and 0 <= s_out < S else None
        exits = [(s_out, slot(s_out))] if last and 0 <= s_out < S else []
        s_exit = i - (L - 1)
        head = (s_exit, slot(s_exit) if last else None) if 0 <= s_exit < S else None
        steps.append(StageStep(nodes, [slot(n.segment) for n in nodes], [n.layer for n in nodes],
                               recv, enter, send, exits, head))
    return StagePlan(rank, world, S, L, blk, n_slots, steps)


def run_stage(plan: StagePlan, backend, comm) -> None:
    """Drive one rank through every global step. ``comm`` has isend(t, dst),
    recv(t, src) and broadcast(t, src) (torch.distributed: NCCL on GPUs, gloo
    in tests). ``backend`` exposes slot_tensor / after_recv / embed / step /
    head_buffer / head.

    Per step: receive (from rank-1) -> embed (rank 0) -> this rank's cells ->
    asynchronous send (to rank+1) -> the deferred vocab-parallel LM head of the
    segment that left layer L-1 on the previous step (broadcast + head GEMM).
    So every rank's point-to-point traffic of a step is posted before that
    step's collective (no cross-rank ordering deadlock), and the head is off
    the path between a rank's cells and the send the next rank waits for.

    Buffer reuse: a slot with a send in flight is never rewritten (by a
    receive or an embed) before that send's ``wait()`` — on NCCL this orders
    the compute stream after the transfer without blocking the host. The
    last rank's exiting slot is read by the head one step after its exit and
    rewritten no earlier than two steps after it (``n_slots`` = layers + 1).
    """
    r, world = plan.rank, plan.world
    pending = None
    sends: dict[int, object] = {}

    def settle(slot):
        work = sends.pop(slot, None)
        if work is not None:
            work.wait()

    for st in plan.steps:
        if st.recv is not None:
            s, slot = st.recv
            settle(slot)
            comm.recv(backend.slot_tensor(slot), r - 1)
            backend.after_recv(slot)
        if st.enter is not None:
            s, slot = st.enter
            settle(slot)
            backend.embed(s, slot)
        if st.nodes:
            backend.step(st.slots, st.layers)
        if st.send is not None:
            s, slot = st.send
            settle(slot)
            sends[slot] = comm.isend(backend.slot_tensor(slot), r + 1)
        if pending is not None:
            _head(backend, comm, pending, world)
        pending = st.head
    if pending is not None:
        _head(backend, comm, pending, world)
    for work in sends.values():
        work.wait()


def _head(backend, comm, h, world) -> None:
    """Vocab-parallel LM head of one exiting segment: the last rank's token
    rows are broadcast to every rank, each computes its vocab block."""
    s, slot = h
    buf = backend.head_buffer(slot)
    if world > 1:
        comm.broadcast(buf, world - 1)
    backend.head(s, buf)


class TorchP2P:
    """Point-to-point activation hand-off and the LM-head broadcast over
    torch.distributed. NCCL moves device tensors directly (NVLink); under gloo
    (CPU tests, or several ranks sharing one GPU for plumbing checks) device
    tensors are staged through host memory."""

    def __init__(self, dist):
        self.dist = dist
        self.staged = dist.get_backend() == "gloo"

    def _op(self, fn, t, peer, inplace):
        if self.staged and t.is_cuda:
            h = t.detach().to("cpu")
            fn(h, peer)
            if inplace:
                t.copy_(h)
        else:
            fn(t, peer)

    def send(self, t, dst):
        self._op(self.dist.send, t, dst, False)

    def isend(self, t, dst):
        """Asynchronous send; ``.wait()`` on the result before ``t`` is rewritten."""
        if self.staged and t.is_cuda:
            h = t.detach().to("cpu")
            return _Staged(self.dist.isend(h, dst), h)
        return self.dist.isend(t, dst)

    def recv(self, t, src):
        self._op(self.dist.recv, t, src, True)

    def broadcast(self, t, src):
        self._op(lambda x, s: self.dist.broadcast(x, s), t, src, True)

    def all_gather(self, out_list, t):
        if self.staged and t.is_cuda:
            hl = [torch_empty_like_cpu(x) for x in out_list]
            self.dist.all_gather(hl, t.detach().to("cpu"))
            for o, h in zip(out_list, hl):
                o.copy_(h)
        else:
            self.dist.all_gather(out_list, t)

    def all_reduce(self, t):
        self._op(lambda x, _: self.dist.all_reduce(x), t, None, True)


class _Staged:
    """A gloo send handle that keeps its host staging copy alive until waited on."""

    def __init__(self, work, buf):
        self.work, self.buf = work, buf

    def wait(self):
        self.work.wait()
        self.buf = None


def torch_empty_like_cpu(x):
    import torch
    return torch.empty(x.shape, dtype=x.dtype)


# ---------------------------------------------------------------------------
# device backend + session (bench / users on N GPUs)
# ---------------------------------------------------------------------------

class DeviceBackend:
    """CUDA ``Engine`` behind ``run_stage``. With ``graphs`` set, each embed /
    step / head launch sequence is captured once (``mode='capture'``) and then
    replayed as one CUDA graph (``mode='replay'``); the NCCL hand-offs between
    them stay eager."""

    def __init__(self, engine, runner_ids, logits, state, seg: int, stream_fn, vocab: range | None = None,
                 head_in=None, lse=None):
        self.e = engine
        self.ids = runner_ids
        self.logits = logits
        self.state = state
        self.seg = seg
        self.stream = stream_fn
        V = engine.cfg.vocab_size
        self.vocab = vocab if vocab is not None else range(0, V)
        self.head_in = head_in
        self.lse = lse
        self.mode = "eager"
        self.graphs: dict = {}
        self.step_no = 0

    def _run(self, key, fn):
        import torch
        if self.mode == "eager":
            fn()
        elif self.mode == "capture":
            if key in self.graphs:
                return   # same launch sequence as an earlier step (same slots / layers): one graph serves both
            g = torch.cuda.CUDAGraph()
            if getattr(self, "_cap_stream", None) is None:
                self._cap_stream = torch.cuda.Stream()   # one capture stream for every step graph
            side = self._cap_stream
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    fn()
            torch.cuda.current_stream().wait_stream(side)
            self.graphs[key] = g
        else:
            self.graphs[key].replay()

    def slot_tensor(self, slot):
        return self.e.xs[slot]

    def after_recv(self, slot):
        from . import _lib
        if self.e.xs_bf is not None:
            x = self.e.xs[slot]
            self._run(("cast", slot), lambda: _lib.check(_lib.load().armt_cast(
                x.data_ptr(), _lib.F32, self.e.xs_bf[slot].data_ptr(), _lib.BF16, x.numel(), self.stream()), "cast"))

    def embed(self, s, slot):
        self._run(("embed", s), lambda: self.e.embed(self.ids[s * self.seg:(s + 1) * self.seg], slot, self.stream()))

    def step(self, slots, layers):
        self._run(("step", tuple(slots), tuple(layers)),
                  lambda: self.e.step(slots, layers, self.state, self.stream()))

    def head_buffer(self, slot):
        """Token rows of the exiting segment: the last rank's slot (bf16 copy), or
        this rank's receive buffer for the broadcast."""
        if slot is not None:
            return self.e.xs_bf[slot][:self.seg]
        return self.head_in

    def head(self, s, buf):
        v0, v1 = self.vocab.start, self.vocab.stop
        if v1 <= v0:
            return
        ptr, ld = buf.data_ptr(), buf.shape[-1]
        if self.lse is not None:
            self._run(("head", s, ptr), lambda: self.e.unembed_block(ptr, ld, v0, v1, s * self.seg, self.stream(),
                                                                   lse=self.lse))
        else:
            self._run(("head", s, ptr), lambda: self.e.unembed_block(ptr, ld, v0, v1, s * self.seg, self.stream(),
                                                                   out=self.logits))

    # single-rank compatibility (tests/test_gpu_sharded.py drives stages by hand)
    def unembed(self, s, slot):
        self.head(s, self.head_buffer(slot))


class ShardedSession:
    """Session (executors.Session API) for one rank of a layer-sharded run.

    ``forward`` returns this rank's vocab block of the logits (vocab-parallel
    LM head; ``vocab`` is the block); a ``scoring`` session keeps only the
    fused next-token NLL partials and ``nll`` returns the full per-token NLL
    on every rank (one all-gather of per-row (max, sum) pairs + one
    all-reduce of the target logits)."""

    def __init__(self, weights, cfg, n_tokens: int, rank: int, world: int, device=None,
                 schedule: str = "diagonal", scoring: bool = False, graphs: bool = True):
        import torch
        import torch.distributed as dist
        from .engine import Engine, MemoryState, prepare_weights
        if schedule != "diagonal":
            raise InputError("layer sharding pipelines the diagonal schedule only")
        self.cfg, self.n, self.rank, self.world = cfg, int(n_tokens), rank, world
        S = -(-self.n // cfg.segment_size)
        seg = cfg.segment_size
        self.plan = stage_plan(S, cfg.n_layers, rank, world)
        blk = self.plan.layers
        self.vocab = vocab_blocks(cfg.vocab_size, world)[rank]
        # this rank's layers, its vocab block of the unembedding, the embedding only on stage 0
        self.p = prepare_weights(weights, "bf16", device, layers=blk, vocab=self.vocab, embedding=blk.start == 0)
        dev = self.p.device
        self.engine = Engine(self.p, self.plan.max_members, self.plan.n_slots)
        self.state = MemoryState.fresh(cfg, dev, n_layers=len(blk))
        self.ids = torch.zeros(S * seg, dtype=torch.int64, device=dev)
        nv = len(self.vocab)
        self.scoring = scoring
        self.logits = None
        lse = None
        if scoring:
            tiles = max(1, -(-nv // 256))
            self.lse_part = torch.empty(S * seg, tiles, 2, device=dev)
            self.lse_tgt = torch.zeros(S * seg, device=dev)
            self.ids_local = torch.zeros(S * seg, dtype=torch.int64, device=dev)
            lse = (self.lse_part, self.lse_tgt, self.ids_local, self.n)
            self.row_ms = torch.empty(S * seg, 2, device=dev)
        else:
            self.logits = torch.empty(S * seg, nv, dtype=torch.bfloat16, device=dev)
        self.head_in = torch.empty(seg, cfg.d_model, dtype=torch.bfloat16, device=dev)
        self.nll_rows = torch.empty(max(self.n - 1, 1), device=dev)
        self.backend = DeviceBackend(self.engine, self.ids, self.logits, self.state, seg,
                                     lambda: torch.cuda.current_stream().cuda_stream, vocab=self.vocab,
                                     head_in=self.head_in, lse=lse)
        self.comm = TorchP2P(dist) if world > 1 else None
        self.use_graphs = graphs
        self.kernels_per_forward = None

        class _R:  # bench compatibility: sess.runner.engine
            pass
        self.runner = _R()
        self.runner.engine = self.engine

    def _load_ids(self, tokens):
        import torch
        from .executors import check_ids
        t = torch.as_tensor(tokens).reshape(-1).to(self.ids.device)
        if t.numel() != self.n:
            raise InputError(f"session compiled for {self.n} tokens, got {t.numel()}")
        check_ids(t, self.cfg.vocab_size)
        self.ids[:self.n].copy_(t, non_blocking=True)
        if self.n < self.ids.numel():
            self.ids[self.n:].zero_()
        if self.scoring:
            torch.sub(self.ids, self.vocab.start, out=self.ids_local)

    def _forward(self):
        self.state.A.zero_()
        self.state.z.zero_()
        if self.state.memop is None:
            self.state.sync_shadow(self.p)
        else:
            self.state.memop.zero_()   # bf16x3 split of the zero state
        if self.scoring:
            self.lse_tgt.zero_()
        run_stage(self.plan, self.backend, self.comm)

    def warm_eager(self):
        import torch
        from . import _lib
        self.backend.mode = "eager"
        before = _lib.kernel_count()
        self._forward()
        torch.cuda.synchronize()
        self.kernels_per_forward = _lib.kernel_count() - before

    def capture(self):
        """Capture every embed / step / head launch sequence as its own CUDA graph
        (the capture pass executes nothing; NCCL hand-offs stay eager)."""
        import torch
        if not self.use_graphs:
            return
        self.backend.mode = "capture"
        self._forward()
        torch.cuda.synchronize()
        self.backend.mode = "replay"

    def warm(self):
        self.warm_eager()
        self.capture()

    def forward(self, tokens=None):
        if tokens is not None:
            self._load_ids(tokens)
        self._forward()
        return self.logits[:self.n] if self.logits is not None else None

    def nll(self, tokens=None):
        """Per-token next-token NLL (n-1 values, device) on every rank."""
        import torch
        from . import _lib
        if not self.scoring:
            raise InputError("the sharded path scores through a scoring=True session (vocab-parallel NLL)")
        self.forward(tokens)
        lib = _lib.load()
        st = torch.cuda.current_stream().cuda_stream
        rows = self.n - 1
        tiles = self.lse_part.shape[1]
        if len(self.vocab):
            _lib.check(lib.armt_lse_reduce(self.lse_part.data_ptr(), tiles, tiles, self.row_ms.data_ptr(), rows,
                                           st), "lse_reduce")
        else:  # empty vocab block (more ranks than 256-column tiles): neutral partials
            self.row_ms[:, 0].fill_(float("-inf"))
            self.row_ms[:, 1].zero_()
        if self.world > 1:
            parts = [torch.empty_like(self.row_ms) for _ in range(self.world)]
            self.comm.all_gather(parts, self.row_ms)
            ms = torch.stack(parts, 1).contiguous()           # (rows, ranks, 2)
            tgt = self.lse_tgt.clone()
            self.comm.all_reduce(tgt)                         # exactly one rank holds each target logit
        else:
            ms, tgt = self.row_ms[:, None, :].contiguous(), self.lse_tgt
        _lib.check(lib.armt_lse_finalize(ms.data_ptr(), self.world, self.world, tgt.data_ptr(),
                                         self.ids.data_ptr() + 8, self.nll_rows.data_ptr(), rows, st),
                   "lse_finalize")
        return self.nll_rows[:rows]
