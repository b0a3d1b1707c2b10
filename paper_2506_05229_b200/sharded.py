"""Layer-sharded (pipeline-over-the-wavefront) execution on 1..N GPUs.

SURVEY §8(e): the diagonal wavefront shards naturally by layer. Rank r owns
the contiguous layer block [lo_r, hi_r) — its weights and its fp32 memory
state (A, z never move). At global step i it runs the cells {(i-l, l) :
l in [lo_r, hi_r)} as one grouped step. The only cross-rank edge is
(s, lo_r - 1) -> (s, lo_r): after step i-1 rank r-1 sends the activation of
segment s = i - lo_r (its last layer's output, T x d fp32) and rank r receives
it before step i. Rank 0 embeds; the last rank runs the LM head.

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
    exits: list[tuple[int, int]]   # (segment, slot) unembedded after the step (last rank)


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
    n_slots = max(1, min(S, hi - lo))
    steps = []
    for i in range(S + L - 1):
        nodes = [n for n in diagonal_members(i, S, L) if lo <= n.layer < hi]
        slot = lambda s: s % n_slots  # noqa: E731
        s_in = i - lo
        recv = (s_in, slot(s_in)) if lo > 0 and 0 <= s_in < S else None
        enter = (i, slot(i)) if lo == 0 and i < S else None
        s_out = i - (hi - 1)
        send = (s_out, slot(s_out)) if hi < L and 0 <= s_out < S else None
        exits = [(s_out, slot(s_out))] if hi == L and 0 <= s_out < S else []
        steps.append(StageStep(nodes, [slot(n.segment) for n in nodes], [n.layer for n in nodes],
                               recv, enter, send, exits))
    return StagePlan(rank, world, S, L, blk, n_slots, steps)


def run_stage(plan: StagePlan, backend, comm) -> None:
    """Drive one rank through every global step. ``comm`` has send(t, dst)
    and recv(t, src) (torch.distributed P2P: NCCL on GPUs, gloo in tests)."""
    r = plan.rank
    for st in plan.steps:
        if st.recv is not None:
            s, slot = st.recv
            comm.recv(backend.slot_tensor(slot), r - 1)
            backend.after_recv(slot)
        if st.enter is not None:
            s, slot = st.enter
            backend.embed(s, slot)
        if st.nodes:
            backend.step(st.slots, st.layers)
        if st.send is not None:
            s, slot = st.send
            comm.send(backend.slot_tensor(slot), r + 1)
        for s, slot in st.exits:
            backend.unembed(s, slot)


class TorchP2P:
    """Point-to-point activation hand-off over torch.distributed."""

    def __init__(self, dist):
        self.dist = dist

    def send(self, t, dst):
        self.dist.send(t, dst)

    def recv(self, t, src):
        self.dist.recv(t, src)


# ---------------------------------------------------------------------------
# device backend + session (bench / users on N GPUs)
# ---------------------------------------------------------------------------

class DeviceBackend:
    def __init__(self, engine, runner_ids, logits, state, seg: int, stream_fn):
        self.e = engine
        self.ids = runner_ids
        self.logits = logits
        self.state = state
        self.seg = seg
        self.stream = stream_fn

    def slot_tensor(self, slot):
        return self.e.xs[slot]

    def after_recv(self, slot):
        from . import _lib
        if self.e.xs_bf is not None:
            x = self.e.xs[slot]
            _lib.check(_lib.load().armt_cast(x.data_ptr(), _lib.F32, self.e.xs_bf[slot].data_ptr(), _lib.BF16,
                                             x.numel(), self.stream()), "cast")

    def embed(self, s, slot):
        self.e.embed(self.ids[s * self.seg:(s + 1) * self.seg], slot, self.stream())

    def step(self, slots, layers):
        self.e.step(slots, layers, self.state, self.stream())

    def unembed(self, s, slot):
        self.e.unembed(slot, self.logits, s * self.seg, self.stream())


class ShardedSession:
    """Session (executors.Session API) for one rank of a layer-sharded run."""

    def __init__(self, weights, cfg, n_tokens: int, rank: int, world: int, device=None,
                 schedule: str = "diagonal"):
        import torch
        import torch.distributed as dist
        from .engine import Engine, MemoryState, prepare_weights
        if schedule != "diagonal":
            raise InputError("layer sharding pipelines the diagonal schedule only")
        self.cfg, self.n, self.rank, self.world = cfg, int(n_tokens), rank, world
        S = -(-self.n // cfg.segment_size)
        self.plan = stage_plan(S, cfg.n_layers, rank, world)
        blk = self.plan.layers
        self.p = prepare_weights(weights, "bf16", device, layers=blk)
        dev = self.p.device
        self.engine = Engine(self.p, self.plan.max_members, self.plan.n_slots)
        self.state = MemoryState.fresh(cfg, dev, n_layers=len(blk))
        self.ids = torch.zeros(S * cfg.segment_size, dtype=torch.int64, device=dev)
        last = rank == world - 1
        self.logits = (torch.empty(S * cfg.segment_size, cfg.vocab_size, dtype=torch.bfloat16, device=dev)
                       if last else None)
        self.nll_rows = torch.empty(max(self.n - 1, 1), device=dev) if last else None
        self.backend = DeviceBackend(self.engine, self.ids, self.logits, self.state, cfg.segment_size,
                                     lambda: torch.cuda.current_stream().cuda_stream)
        self.comm = TorchP2P(dist)
        self.kernels_per_forward = None

        class _R:  # bench compatibility: sess.runner.engine
            pass
        self.runner = _R()
        self.runner.engine = self.engine

    def _load_ids(self, tokens):
        import torch
        self.ids[:self.n].copy_(torch.as_tensor(tokens).reshape(-1).to(self.ids.device), non_blocking=True)

    def _forward(self):
        self.state.A.zero_()
        self.state.z.zero_()
        self.state.sync_shadow(self.p)
        run_stage(self.plan, self.backend, self.comm)

    def warm_eager(self):
        import torch
        from . import _lib
        before = _lib.kernel_count()
        self._forward()
        torch.cuda.synchronize()
        self.kernels_per_forward = _lib.kernel_count() - before

    def capture(self):
        """P2P hand-offs stay eager (NCCL send/recv per step); nothing to capture."""

    def forward(self, tokens=None):
        if tokens is not None:
            self._load_ids(tokens)
        self._forward()
        return None if self.logits is None else self.logits[:self.n]

    def nll(self, tokens=None):
        import torch
        from . import _lib
        logits = self.forward(tokens)
        if logits is None:
            return None
        _lib.check(_lib.load().armt_logits_nll(logits.data_ptr(), _lib.BF16, self.cfg.vocab_size,
                                               self.ids[1:self.n].data_ptr(), self.nll_rows.data_ptr(), self.n - 1,
                                               self.cfg.vocab_size, torch.cuda.current_stream().cuda_stream), "nll")
        return self.nll_rows[:self.n - 1]
