"""Per-core public API over device tensors (mirrors armt/layers.py and
armt/memory.py entry points).

These are the reference's stacked cores with the reference's signatures —
``retrieve_stack(state, layers, x, prepared)``, ``forward_stack(prepared,
layers, x)``, ``update_stack(state, layers, mem_out, prepared)`` — taking
(G, T, d) float32 device tensors. Each call stages the members into an
Engine's activation slots and runs the same grouped kernels the executors
use, so "grouped equals looped" holds bitwise here as it does in the
reference (armt/layers.py:1-9).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import Engine, MemoryState, PreparedWeights
from .errors import DimensionError, InputError, SchedulingError


@dataclass
class SegmentActivation:
    """[tokens_part; mem_part] of one in-flight segment (armt/layers.py:28-47)."""

    data: torch.Tensor          # (T, d) float32, on device
    n_token_rows: int
    segment_index: int
    layer_cursor: int = 0

    @property
    def tokens_part(self) -> torch.Tensor:
        return self.data[:self.n_token_rows]

    @property
    def mem_part(self) -> torch.Tensor:
        return self.data[self.n_token_rows:]


def _engine(prepared: PreparedWeights, G: int) -> Engine:
    cache = prepared.__dict__.setdefault("_engines", {})
    eng = cache.get(G)
    if eng is None:
        # the per-core API runs forward_stack without a preceding retrieve epilogue,
        # so it uses the stand-alone RMSNorm rather than the fused row statistics
        eng = Engine(prepared, G, G, fused_norm=False)
        cache[G] = eng
    return eng


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _stage(eng: Engine, x: torch.Tensor, rows: slice | None = None) -> None:
    G = x.shape[0]
    dst = eng.xs[:G] if rows is None else eng.xs[:G, rows]
    dst.copy_(x)
    if eng.xs_bf is not None:
        dstb = eng.xs_bf[:G] if rows is None else eng.xs_bf[:G, rows]
        dstb.copy_(dst)


def _check_stack(prepared: PreparedWeights, layers, x: torch.Tensor, rows: int) -> list[int]:
    cfg = prepared.config
    if not isinstance(x, torch.Tensor) or x.dim() != 3:
        raise DimensionError("x must be a (G, T, d) tensor")
    if x.shape[1:] != (rows, cfg.d_model):
        raise DimensionError(f"x members must be {(rows, cfg.d_model)}, got {tuple(x.shape[1:])}")
    if x.dtype != torch.float32 or x.device != prepared.device:
        raise DimensionError("x must be float32 on the weights' device")
    layers = [int(l) for l in np.asarray(layers).reshape(-1)]
    if len(layers) != x.shape[0]:
        raise DimensionError(f"{len(layers)} layers for {x.shape[0]} members")
    if not layers:
        raise SchedulingError("grouped call needs at least one member")
    for l in layers:
        if not 0 <= l < cfg.n_layers:
            raise SchedulingError(f"layer index {l} out of range 0..{cfg.n_layers - 1}")
    return layers


def retrieve_stack(state: MemoryState, layers, x: torch.Tensor, prepared: PreparedWeights,
                   pool=None) -> torch.Tensor:
    """x + guarded associative readout per member (armt/memory.py:132-152)."""
    layers = _check_stack(prepared, layers, x, prepared.T)
    state.check_compatible(prepared)
    G = len(layers)
    eng = _engine(prepared, G)
    _stage(eng, x)
    state.sync_shadow(prepared)
    eng.retrieve(list(range(G)), layers, state, _stream())
    return eng.xs[:G].clone()


def forward_stack(prepared: PreparedWeights, layers, x: torch.Tensor, pool=None) -> torch.Tensor:
    """Pre-norm block for G members (armt/layers.py:235-246)."""
    layers = _check_stack(prepared, layers, x, prepared.T)
    G = len(layers)
    eng = _engine(prepared, G)
    _stage(eng, x)
    eng.forward(list(range(G)), layers, _stream())
    return eng.xs[:G].clone()


def update_stack(state: MemoryState, layers, mem_out: torch.Tensor, prepared: PreparedWeights,
                 pool=None) -> None:
    """Delta-rule fold of each member's memory rows (armt/memory.py:155-180)."""
    cfg = prepared.config
    layers = _check_stack(prepared, layers, mem_out, cfg.num_mem_tokens)
    if len(set(layers)) != len(layers):
        raise SchedulingError(f"duplicate layer index in group: {sorted(layers)}")
    state.check_compatible(prepared)
    G = len(layers)
    eng = _engine(prepared, G)
    _stage(eng, mem_out, slice(cfg.segment_size, prepared.T))
    state.sync_shadow(prepared)
    eng.update(list(range(G)), layers, state, _stream())
    for l in layers:
        state.updates[l] += 1


def dpfp(x: torch.Tensor, nu: int) -> torch.Tensor:
    """DPFP feature map on the device (armt/memory.py:34-45): (..., m) -> (..., 2*nu*m)."""
    if nu < 1:
        raise InputError(f"dpfp order must be >= 1, got {nu}")
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise DimensionError("dpfp expects a CUDA tensor")
    m = x.shape[-1]
    rows = x.numel() // m
    q = x.reshape(1, rows, m).float().contiguous()
    phi = torch.empty(1, rows, 2 * nu * m, device=x.device)
    den = torch.empty(1, rows, device=x.device)
    z = torch.zeros(1, 2 * nu * m, device=x.device)
    mem = _lib.members([0], [0])
    _lib.check(_lib.load().armt_dpfp_den(mem, q.data_ptr(), rows * m, z.data_ptr(), phi.data_ptr(), _lib.F32,
                                         2 * nu * m, rows * 2 * nu * m, den.data_ptr(), rows, rows, m, nu,
                                         _stream()), "dpfp")
    return phi.reshape(*x.shape[:-1], 2 * nu * m)


# ---------------------------------------------------------------- single ops

def _check_members(prepared: PreparedWeights, members) -> list[int]:
    """armt/layers.py:253-278."""
    if not members:
        raise SchedulingError("grouped forward needs at least one member")
    L = prepared.config.n_layers
    if len(members) > L:
        raise SchedulingError(f"group of {len(members)} exceeds layer count {L}")
    layers = []
    for l, act in members:
        if not 0 <= l < L:
            raise SchedulingError(f"layer index {l} out of range 0..{L - 1}")
        if act.layer_cursor != l:
            raise SchedulingError(f"segment {act.segment_index} is at layer {act.layer_cursor}, not {l}")
        if tuple(act.data.shape) != (prepared.T, prepared.config.d_model):
            raise DimensionError(f"segment {act.segment_index} activation has shape {tuple(act.data.shape)}")
        layers.append(l)
    if len(set(layers)) != len(layers):
        raise SchedulingError(f"duplicate layer index in group: {sorted(layers)}")
    return layers


def grouped_layer_forward(prepared: PreparedWeights, members, pool=None) -> list[SegmentActivation]:
    layers = _check_members(prepared, members)
    y = forward_stack(prepared, layers, torch.stack([a.data for _, a in members]))
    return [SegmentActivation(y[g], a.n_token_rows, a.segment_index, l + 1)
            for g, (l, a) in enumerate(members)]


def layer_forward(prepared: PreparedWeights, layer: int, activation: SegmentActivation,
                  pool=None) -> SegmentActivation:
    return grouped_layer_forward(prepared, [(layer, activation)])[0]


def assoc_retrieve(state: MemoryState, layer: int, activation: SegmentActivation,
                   prepared: PreparedWeights) -> SegmentActivation:
    """armt/memory.py:193-202."""
    if not 0 <= layer < prepared.config.n_layers:
        raise InputError(f"layer index {layer} out of range 0..{prepared.config.n_layers - 1}")
    y = retrieve_stack(state, [layer], activation.data[None], prepared)
    return SegmentActivation(y[0], activation.n_token_rows, activation.segment_index, activation.layer_cursor)


def assoc_update(state: MemoryState, layer: int, mem_out: torch.Tensor, prepared: PreparedWeights) -> None:
    """armt/memory.py:205-215."""
    cfg = prepared.config
    if not 0 <= layer < cfg.n_layers:
        raise InputError(f"layer index {layer} out of range 0..{cfg.n_layers - 1}")
    if mem_out.dim() != 2 or tuple(mem_out.shape) != (cfg.num_mem_tokens, cfg.d_model):
        raise DimensionError(f"memory-token outputs must be {(cfg.num_mem_tokens, cfg.d_model)}, "
                             f"got {tuple(mem_out.shape)}")
    update_stack(state, [layer], mem_out.contiguous()[None], prepared)


def embed_segment(prepared: PreparedWeights, token_ids, segment_index: int) -> SegmentActivation:
    """armt/layers.py:306-318."""
    cfg = prepared.config
    ids = torch.as_tensor(np.asarray(token_ids, dtype=np.int64))
    if ids.dim() != 1 or ids.shape[0] != cfg.segment_size:
        raise InputError(f"segment must hold exactly {cfg.segment_size} token ids, got {tuple(ids.shape)}")
    if ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= cfg.vocab_size):
        raise InputError(f"token ids must lie in [0, {cfg.vocab_size})")
    eng = _engine(prepared, 1)
    eng.embed(ids.to(prepared.device), 0, _stream())
    return SegmentActivation(eng.xs[0].clone(), cfg.segment_size, segment_index, 0)


def unembed(prepared: PreparedWeights, activation: SegmentActivation) -> torch.Tensor:
    """Logits for the token rows, no final norm (armt/layers.py:321-323)."""
    cfg = prepared.config
    eng = _engine(prepared, 1)
    _stage(eng, activation.data[None])
    dt = torch.bfloat16 if prepared.dtype_name == "bf16" else torch.float32
    out = torch.empty(cfg.segment_size, cfg.vocab_size, dtype=dt, device=prepared.device)
    eng.unembed(0, out, 0, _stream())
    return out
