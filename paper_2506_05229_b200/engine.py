"""Device-resident weights, memory state and the per-step kernel sequence.

``Engine.step`` is the B200 replacement for one pass of the reference's
stacked cores (armt/executors.py:200-203): retrieve_stack -> forward_stack ->
update_stack for G (slot, layer) members in ONE grouped launch per op. The
executors (``executors.py``) drive it along the wavefront; the public
per-core functions (``memory.py``, ``layers.py``) are thin wrappers.

HBM layout
  weights   K-major (out, in) per layer, layer-stacked, bf16 (or f32 in the
            parity mode): wqkv (L, 3d, d), wo (L, d, d), wgu (L, 2F, d) with
            gate/up interleaved in blocks of ``swiglu_block`` columns, wdown
            (L, d, F), wqa (L, d_mem, d), wkvb (L, Nkvb, d) = [W_v; W_k; W_beta; 0],
            unemb (V, d). F = d_ff padded to a multiple of 32 (zero rows/cols).
  state     A (L, d, d_phi) f32, z (L, d_phi) f32 — the reference MemoryState
            shapes — plus (bf16 mode) the memory operand ``memop`` (L, NB, 2P),
            P = d_phi rounded up to 32: per layer the [hi|lo] bf16 split of A
            (rows 0..d-1) and of z (row d); the tensor-core fold reads it as a
            bf16x3 operand (hi re-read as the third part through a K wrap),
            retrieval reads its hi part. Refreshed by the fold.
  slots     residual stream per in-flight segment: xs (n_slots, T, d) f32 and,
            in bf16 mode, its bf16 copy xs_bf written by the same epilogues.
  members   per-step temporaries stacked over members: h, qkv, ctx, gu, q, phi,
            den, kvb.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import BF16, F32, EPI_RESIDUAL, EPI_RETRIEVE, EPI_ROPE, EPI_STORE, EPI_SWIGLU
from .config import ModelConfig, ROPE_BASE, resolve_dtype
from .errors import DimensionError, InputError
from .weights import GroupedWeights, expected_shapes


# bf16 path: DPFP + phi.z fused into the q-projection epilogue (ARMT_FUSED_DPFP=0: two launches)
FUSED_DPFP = __import__("os").environ.get("ARMT_FUSED_DPFP", "1") == "1"


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


# ============================================================================
# Prepared weights
# ============================================================================

@dataclass
class PreparedWeights:
    """Device weights in kernel layouts (armt/layers.py:54-134 counterpart)."""

    config: ModelConfig
    dtype_name: str
    eps_assoc: float
    device: torch.device
    wdtype: torch.dtype
    T: int
    d_head: int
    d_phi: int
    d_phi_pad: int
    d_ff_pad: int
    swiglu_block: int
    n_kvb: int
    embedding: torch.Tensor
    mem_embedding: torch.Tensor
    wqkv: torch.Tensor
    wo: torch.Tensor
    wgu: torch.Tensor
    wdown: torch.Tensor
    attn_gain: torch.Tensor       # (folded into wqkv / wgu; kept for inspection)
    mlp_gain: torch.Tensor
    unit_gain: torch.Tensor       # ones: the stand-alone RMSNorm applies no gain (it is in the weights)
    wqa: torch.Tensor
    wkvb: torch.Tensor
    unemb: torch.Tensor
    rope_cos: torch.Tensor        # (T, d_head/2): stand-alone RoPE kernel (f32 mode)
    rope_sin: torch.Tensor
    rope_cos_t: torch.Tensor      # (d_head/2, T): fused QKV epilogue (bf16 mode)
    rope_sin_t: torch.Tensor
    layer_base: int = 0
    vocab_base: int = 0            # first unembedding column held (vocab-parallel head)

    @property
    def ab(self) -> int:
        return BF16 if self.dtype_name == "bf16" else F32

    @property
    def v_off(self) -> int:
        return 0

    @property
    def k_off(self) -> int:
        return self.config.d_model

    @property
    def b_off(self) -> int:
        return self.config.d_model + self.config.d_mem


def prepare_weights(weights: GroupedWeights, dtype_name: str = "bf16", device=None,
                    layers: range | None = None, vocab: range | None = None,
                    embedding: bool = True) -> PreparedWeights:
    """Cast, transpose to K-major, pad and upload (one-time setup).

    ``layers`` restricts the per-layer tensors to a contiguous block (layer
    sharding); layer indices stay global in the executors and are rebased here.
    ``vocab`` uploads only that block of unembedding columns (vocab-parallel
    LM head; ``vocab_base`` records its start) and ``embedding=False`` skips
    the token embedding (pipeline stages other than the first).
    """
    cfg = weights.config
    resolve_dtype(dtype_name)
    for name, shape in expected_shapes(cfg).items():
        got = tuple(getattr(weights, name).shape)
        if tuple(got) != shape:
            raise InputError(f"weight tensor {name!r} has shape {got}, config expects {shape}")
    if not torch.cuda.is_available():
        from .errors import DeviceError
        raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    bf16 = dtype_name == "bf16"
    wdt = torch.bfloat16 if bf16 else torch.float32
    L, d, dff, dm = cfg.n_layers, cfg.d_model, cfg.d_ff, cfg.d_mem
    lo, hi = (0, L) if layers is None else (layers.start, layers.stop)
    if bf16 and d % 8:
        raise DimensionError("bf16 path needs d_model % 8 == 0 (TMA 16-byte rows)")
    dh = cfg.d_head
    T = cfg.tokens_per_segment
    d_phi = cfg.d_phi
    d_phi_pad = _round_up(d_phi, 32) if bf16 else d_phi   # [hi | lo] memory operand wraps at 2P (64-col K blocks)
    d_ff_pad = _round_up(dff, 32)
    block = 128 if d_ff_pad % 128 == 0 else 32
    n_kvb = _round_up(d + dm + 1, 16)

    def up(name, sl=True):
        a = getattr(weights, name)
        a = a[lo:hi] if sl else a
        if isinstance(a, torch.Tensor):
            return a.to(dev, torch.float32).contiguous()
        return torch.as_tensor(np.ascontiguousarray(a)).to(dev, torch.float32)

    def kmajor(t):  # (L, in, out) -> (L, out, in)
        return t.transpose(1, 2).contiguous()

    # RMSNorm gains fold into the consuming weights: (x/r * g) @ W = (x/r) @ (diag(g) W)
    g_attn, g_mlp = up("attn_gain"), up("mlp_gain")
    wqkv = kmajor(torch.cat([up("wq"), up("wk"), up("wv")], dim=2) * g_attn[:, :, None]).to(wdt)
    wo = kmajor(up("wo")).to(wdt)
    Ls = hi - lo
    gate = torch.zeros(Ls, d, d_ff_pad, device=dev)
    upw = torch.zeros(Ls, d, d_ff_pad, device=dev)
    gate[:, :, :dff] = up("w_gate") * g_mlp[:, :, None]
    upw[:, :, :dff] = up("w_in") * g_mlp[:, :, None]
    nt = d_ff_pad // block
    gu = torch.stack([gate.view(Ls, d, nt, block), upw.view(Ls, d, nt, block)], dim=3)
    wgu = kmajor(gu.reshape(Ls, d, 2 * d_ff_pad)).to(wdt)
    del gate, upw, gu
    wout = torch.zeros(Ls, d_ff_pad, d, device=dev)
    wout[:, :dff] = up("w_out")
    wdown = kmajor(wout).to(wdt)
    del wout
    wkvb = torch.zeros(Ls, n_kvb, d, device=dev)
    wkvb[:, :d] = up("w_v_mem")
    wkvb[:, d:d + dm] = up("w_k_mem")
    wkvb[:, d + dm] = up("w_beta")[:, 0]
    inv = ROPE_BASE ** (-np.arange(0, dh, 2, dtype=np.float64) / dh)
    ang = np.arange(T, dtype=np.float64)[:, None] * inv[None, :]
    prepared = PreparedWeights(
        config=cfg, dtype_name=dtype_name, eps_assoc=cfg.effective_eps_assoc(dtype_name),
        device=dev, wdtype=wdt, T=T, d_head=dh, d_phi=d_phi, d_phi_pad=d_phi_pad,
        d_ff_pad=d_ff_pad, swiglu_block=block, n_kvb=n_kvb,
        embedding=(up("embedding", False).to(wdt) if embedding
                   else torch.zeros(0, d, dtype=wdt, device=dev)),
        mem_embedding=up("mem_embedding", False).to(wdt),
        wqkv=wqkv, wo=wo, wgu=wgu, wdown=wdown,
        attn_gain=g_attn.contiguous(), mlp_gain=g_mlp.contiguous(),
        unit_gain=torch.ones_like(g_attn).contiguous(),
        wqa=up("w_q_assoc").to(wdt).contiguous(), wkvb=wkvb.to(wdt),
        unemb=_unemb(weights.unembedding, vocab, dev, wdt),
        rope_cos=torch.as_tensor(np.cos(ang), dtype=torch.float32).to(dev).contiguous(),
        rope_sin=torch.as_tensor(np.sin(ang), dtype=torch.float32).to(dev).contiguous(),
        rope_cos_t=torch.as_tensor(np.cos(ang).T, dtype=torch.float32).to(dev).contiguous(),
        rope_sin_t=torch.as_tensor(np.sin(ang).T, dtype=torch.float32).to(dev).contiguous(),
    )
    prepared.layer_base = lo
    prepared.vocab_base = 0 if vocab is None else vocab.start
    torch.cuda.synchronize(dev)
    return prepared


def _unemb(u, vocab: range | None, dev, wdt) -> torch.Tensor:
    """(V, d) K-major unembedding (or its [v0, v1) row block), uploaded column
    block by column block so the host never materialises a second full copy."""
    V = u.shape[1]
    v0, v1 = (0, V) if vocab is None else (vocab.start, vocab.stop)
    out = torch.empty(v1 - v0, u.shape[0], dtype=wdt, device=dev)
    step = 16384
    for a in range(v0, v1, step):
        b = min(v1, a + step)
        blk = u[:, a:b]
        t = blk if isinstance(blk, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(blk))
        out[a - v0:b - v0] = t.to(dev, torch.float32).t().to(wdt)
    return out


# ============================================================================
# Memory state
# ============================================================================

@dataclass
class MemoryState:
    """Per-layer fast weights on device (armt/memory.py:52-87).

    A (L, d, d_phi) f32, z (L, d_phi) f32 (fp32 in both device precisions),
    updates (L,) int64 on the host (pure bookkeeping). ``memop`` (bf16 mode)
    is derived state: the bf16x3 split of A and z read by the tensor-core
    retrieval and fold (see engine module docstring).
    """

    A: torch.Tensor
    z: torch.Tensor
    updates: np.ndarray
    memop: torch.Tensor | None = field(default=None, repr=False)

    @classmethod
    def fresh(cls, config: ModelConfig, device=None, n_layers: int | None = None) -> "MemoryState":
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        L = config.n_layers if n_layers is None else n_layers
        return cls(A=torch.zeros(L, config.d_model, config.d_phi, device=dev),
                   z=torch.zeros(L, config.d_phi, device=dev),
                   updates=np.zeros(L, np.int64))

    @classmethod
    def from_numpy(cls, A, z, updates, device=None) -> "MemoryState":
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        return cls(A=torch.as_tensor(np.asarray(A, np.float32)).to(dev).contiguous(),
                   z=torch.as_tensor(np.asarray(z, np.float32)).to(dev).contiguous(),
                   updates=np.array(updates, np.int64))

    def clone(self) -> "MemoryState":
        return MemoryState(self.A.clone(), self.z.clone(), self.updates.copy())

    def to_numpy(self):
        return self.A.float().cpu().numpy(), self.z.float().cpu().numpy(), self.updates.copy()

    def check_compatible(self, prepared: PreparedWeights, n_layers: int | None = None) -> None:
        cfg = prepared.config
        L = cfg.n_layers if n_layers is None else n_layers
        want = (L, cfg.d_model, cfg.d_phi)
        if tuple(self.A.shape) != want or tuple(self.z.shape) != (L, cfg.d_phi):
            raise InputError(f"memory state shaped {tuple(self.A.shape)}/{tuple(self.z.shape)}, "
                             f"config expects {want}/{(L, cfg.d_phi)}")
        if self.A.dtype != torch.float32 or self.z.dtype != torch.float32:
            raise InputError("memory state must be float32 on the device path")
        if self.A.device != prepared.device:
            raise InputError(f"memory state on {self.A.device}, weights on {prepared.device}")
        if not (self.A.is_contiguous() and self.z.is_contiguous()):
            raise InputError("memory state tensors must be contiguous")

    def sync_shadow(self, prepared: PreparedWeights) -> None:
        """(Re)build the bf16x3 memory operand from A and z (setup work at run
        start, on the current stream; the fold keeps it in sync afterwards)."""
        if prepared.dtype_name != "bf16":
            return
        L, d, dphi = self.A.shape
        P = prepared.d_phi_pad
        nb = int(_lib.load().armt_memop_rows(d, prepared.config.num_mem_tokens))
        if self.memop is None or tuple(self.memop.shape) != (L, nb, 2 * P):
            self.memop = torch.zeros(L, nb, 2 * P, dtype=torch.bfloat16, device=self.A.device)

        def split(x):
            hi = x.to(torch.bfloat16)
            return hi, (x - hi.float()).to(torch.bfloat16)
        for rows, src in ((slice(0, d), self.A), (slice(d, d + 1), self.z[:, None, :])):
            hi, lo = split(src)
            self.memop[:, rows, 0:dphi] = hi
            self.memop[:, rows, P:P + dphi] = lo


# ============================================================================
# Engine: workspace + one wavefront step
# ============================================================================

class Engine:
    """Kernel sequence for one schedule step over G members.

    ``n_slots`` activation slots hold the residual stream of in-flight
    segments; member g of a step is (slots[g], layers[g]). ``layers`` are
    global layer indices; weights/state may hold only a contiguous block
    starting at ``layer_base`` (layer sharding).
    """

    def __init__(self, prepared: PreparedWeights, max_members: int, n_slots: int,
                 n_state_layers: int | None = None, fused_norm: bool = True, slots_from: "Engine | None" = None):
        p = prepared
        cfg = p.config
        self.p = p
        self.cfg = cfg
        self.lib = _lib.load()
        self.max_members = max_members
        self.n_slots = n_slots
        self.layer_base = getattr(p, "layer_base", 0)
        dev = p.device
        T, d, G = p.T, cfg.d_model, max_members
        wdt = p.wdtype
        self.bf16 = p.dtype_name == "bf16"
        if slots_from is not None:   # a second engine over the same activation slots (dual-stream runner)
            self.xs, self.xs_bf = slots_from.xs, slots_from.xs_bf
        else:
            self.xs = torch.zeros(n_slots, T, d, device=dev)
            self.xs_bf = torch.zeros(n_slots, T, d, dtype=torch.bfloat16, device=dev) if self.bf16 else None
        self.h = torch.empty(G, T, d, dtype=wdt, device=dev)
        self.qkv = torch.empty(G, T, 3 * d, dtype=wdt, device=dev)
        self.ctx = torch.empty(G, T, d, dtype=wdt, device=dev)
        self.gu = torch.empty(G, T, p.d_ff_pad, dtype=wdt, device=dev)
        self.gu_full = None if self.bf16 else torch.empty(G, T, 2 * p.d_ff_pad, dtype=wdt, device=dev)
        self.qm = torch.empty(G, T, cfg.d_mem, device=dev)
        self.phi = torch.zeros(G, T, p.d_phi_pad, dtype=wdt, device=dev)
        self.den = torch.empty(G, T, device=dev)
        self.kvb = torch.empty(G, cfg.num_mem_tokens, p.n_kvb, device=dev)
        if self.bf16:
            nb = int(self.lib.armt_fold_tc_workspace_bytes(G, cfg.num_mem_tokens, d, p.d_phi))
        else:
            nb = int(self.lib.armt_fold_workspace_bytes(G, cfg.num_mem_tokens, p.d_phi))
        self.fold_ws = torch.zeros(max(nb, 16) // 4 + 1, device=dev)  # zero padding is part of the contract
        # fused RMSNorm (bf16, full step path): per-row sum of squares produced by the
        # residual epilogues, consumed (and re-zeroed) by the next GEMM's epilogue
        # the QKV epilogue applies RoPE for head sizes {8,16,32,64,128}; other (even) head
        # sizes run QKV with a plain store + the stand-alone RoPE kernel, and then the
        # RMSNorm cannot ride in that epilogue either (armt/layers.py:169-176 allows any even d_head)
        self.rope_fused = self.bf16 and p.d_head in (8, 16, 32, 64, 128)
        self.fused = self.bf16 and fused_norm and self.rope_fused
        self.ssq_np = (d + 63) // 64
        self.ssq_attn = torch.zeros(G, T, self.ssq_np, device=dev)
        self.ssq_mlp = torch.zeros(G, T, self.ssq_np, device=dev)
        self._cache: dict = {}
        self.probe = None   # optional callable(tag, phase) around the gate/up GEMM (bench roofline)

    # -- argument builders (memoised: graphs/eager replays reuse the structs) --
    def _gemm(self, key, fill):
        args = self._cache.get(key)
        if args is None:
            args = _lib.ArmtGemmArgs()
            fill(args)
            self._cache[key] = args
        return args

    def _members(self, slots, layers):
        key = ("mem", tuple(slots), tuple(layers))
        m = self._cache.get(key)
        if m is None:
            m = _lib.members(slots, [l - self.layer_base for l in layers])
            self._cache[key] = m
        return m

    @staticmethod
    def _tables(args, a_slots, b_index, c_slots):
        args.G = len(b_index)
        for g in range(args.G):
            args.a_slot[g] = int(a_slots[g])
            args.b_index[g] = int(b_index[g])
            args.c_slot[g] = int(c_slots[g])

    # -- embedding boundary ---------------------------------------------------
    def embed(self, ids: torch.Tensor, slot: int, stream: int) -> None:
        """armt/layers.py:306-318 into activation slot ``slot``."""
        p, cfg = self.p, self.cfg
        T, d = p.T, cfg.d_model
        if p.embedding.shape[0] != cfg.vocab_size:
            raise InputError("these prepared weights hold no token embedding (prepare_weights(embedding=False))")
        xb = None if self.xs_bf is None else self.xs_bf[slot].data_ptr()
        _lib.check(self.lib.armt_embed(ids.data_ptr(), p.embedding.data_ptr(), p.mem_embedding.data_ptr(),
                                       p.ab, self.xs[slot].data_ptr(), xb, cfg.segment_size,
                                       cfg.num_mem_tokens, d, cfg.vocab_size, stream), "embed")

    # -- the three stacked cores ---------------------------------------------
    def retrieve(self, slots, layers, state: MemoryState, stream: int, state_layers=None) -> None:
        """retrieve_stack (armt/memory.py:132-152), in place on xs[slots].

        ``state_layers`` index the memory state (default: ``layers``); the
        minibatch plan keeps one state block per copy (state layer b*L + l)
        while the weights stay indexed by ``layers``."""
        if state_layers is None:
            state_layers = layers
        p, cfg, lib = self.p, self.cfg, self.lib
        T, d, G = p.T, cfg.d_model, len(layers)
        lrel = [l - self.layer_base for l in layers]
        gid = list(range(G))
        src = self.xs_bf if self.bf16 else self.xs

        srel = [l - self.layer_base for l in state_layers]
        if self.bf16 and FUSED_DPFP and cfg.d_mem in (16, 32, 64) and 1 <= cfg.dpfp_nu <= 3:
            # q-proj with the DPFP feature map + phi.z in its epilogue: phi (bf16) and den
            # straight from the accumulator, no q round trip (armt/memory.py:137-147)
            def fill_qd(a):
                a.M, a.N, a.K, a.ab_dtype = T, cfg.d_mem, d, p.ab
                a.A, a.lda, a.a_stride = src.data_ptr(), d, T * d
                a.B, a.ldb, a.b_stride = p.wqa.data_ptr(), d, cfg.d_mem * d
                a.C, a.ldc, a.c_stride, a.c_dtype = self.phi.data_ptr(), p.d_phi_pad, T * p.d_phi_pad, BF16
                a.epilogue = _lib.EPI_DPFP
                a.den, a.den_stride = self.den.data_ptr(), T
                a.z, a.nu = state.z.data_ptr(), cfg.dpfp_nu
                self._tables(a, slots, lrel, gid)
                for g in range(G):
                    a.e_index[g] = int(srel[g])
            args = self._gemm(("qd", tuple(slots), tuple(layers), tuple(state_layers), state.z.data_ptr()), fill_qd)
            _lib.check(lib.armt_gemm(args, stream), "retrieve q-proj + DPFP")
        else:
            def fill_q(a):
                a.M, a.N, a.K, a.ab_dtype = T, cfg.d_mem, d, p.ab
                a.A, a.lda, a.a_stride = src.data_ptr(), d, T * d
                a.B, a.ldb, a.b_stride = p.wqa.data_ptr(), d, cfg.d_mem * d
                a.C, a.ldc, a.c_stride, a.c_dtype = self.qm.data_ptr(), cfg.d_mem, T * cfg.d_mem, F32
                a.epilogue = EPI_STORE
                self._tables(a, slots, lrel, gid)
            args = self._gemm(("q", tuple(slots), tuple(layers)), fill_q)
            _lib.check(lib.armt_gemm(args, stream), "retrieve q-proj")
            mem = self._members(slots, state_layers)
            _lib.check(lib.armt_dpfp_den(mem, self.qm.data_ptr(), T * cfg.d_mem, state.z.data_ptr(),
                                         self.phi.data_ptr(), p.ab, p.d_phi_pad, T * p.d_phi_pad,
                                         self.den.data_ptr(), T, T, cfg.d_mem, cfg.dpfp_nu, stream), "dpfp_den")
        bmat = state.memop if self.bf16 else state.A
        ld_b = 2 * p.d_phi_pad if self.bf16 else p.d_phi
        nb_rows = state.memop.shape[1] if self.bf16 else d

        def fill_n(a):
            a.M, a.N, a.K, a.ab_dtype = T, d, p.d_phi_pad, p.ab
            a.A, a.lda, a.a_stride = self.phi.data_ptr(), p.d_phi_pad, T * p.d_phi_pad
            a.B, a.ldb, a.b_stride = bmat.data_ptr(), ld_b, nb_rows * ld_b
            a.C, a.ldc, a.c_stride, a.c_dtype = self.xs.data_ptr(), d, T * d, F32
            a.epilogue = EPI_RETRIEVE
            a.R, a.ldr, a.r_stride = self.xs.data_ptr(), d, T * d
            a.den, a.den_stride, a.eps = self.den.data_ptr(), T, p.eps_assoc
            if self.fused:
                a.C2, a.ldc2, a.c2_stride = self.xs_bf.data_ptr(), d, T * d
                a.ssq_out, a.ssq_stride, a.ssq_np = self.ssq_attn.data_ptr(), T * self.ssq_np, self.ssq_np
            self._tables(a, gid, srel, slots)
        args = self._gemm(("num", tuple(slots), tuple(state_layers), bmat.data_ptr()), fill_n)
        _lib.check(lib.armt_gemm(args, stream), "retrieve numerator")

    def forward(self, slots, layers, stream: int) -> None:
        """forward_stack (armt/layers.py:235-246), in place on xs[slots]."""
        p, cfg, lib = self.p, self.cfg, self.lib
        T, d, G = p.T, cfg.d_model, len(layers)
        lrel = [l - self.layer_base for l in layers]
        gid = list(range(G))
        key = (tuple(slots), tuple(layers), self.fused)
        mem = self._members(slots, layers)
        wout = BF16 if self.bf16 else F32
        fused = self.fused
        # attention sub-block: RMSNorm fused into the QKV epilogue (bf16) or stand-alone
        if not fused:
            _lib.check(lib.armt_rmsnorm(mem, self.xs.data_ptr(), T * d, p.unit_gain.data_ptr(), self.h.data_ptr(),
                                        wout, T * d, T, d, cfg.eps_norm, stream), "rmsnorm attn")
        a_in = self.xs_bf if fused else self.h
        a_idx = slots if fused else gid

        def fill_qkv(a):
            a.M, a.N, a.K, a.ab_dtype = T, 3 * d, d, p.ab
            a.A, a.lda, a.a_stride = a_in.data_ptr(), d, T * d
            a.B, a.ldb, a.b_stride = p.wqkv.data_ptr(), d, 3 * d * d
            a.C, a.ldc, a.c_stride, a.c_dtype = self.qkv.data_ptr(), 3 * d, T * 3 * d, wout
            if self.rope_fused:
                a.epilogue = EPI_ROPE
                a.rope_cos, a.rope_sin = p.rope_cos_t.data_ptr(), p.rope_sin_t.data_ptr()
                a.head_dim, a.rope_cols = p.d_head, 2 * d
                if fused:
                    a.ssq_in, a.ssq_stride, a.ssq_np = self.ssq_attn.data_ptr(), T * self.ssq_np, self.ssq_np
                    a.norm_d, a.norm_eps = d, cfg.eps_norm
            else:
                a.epilogue = EPI_STORE
            self._tables(a, a_idx, lrel, gid)
        _lib.check(lib.armt_gemm(self._gemm(("qkv",) + key, fill_qkv), stream), "qkv")
        if not self.rope_fused:
            _lib.check(lib.armt_rope(G, self.qkv.data_ptr(), 3 * d, T * 3 * d, wout, T, cfg.n_heads, p.d_head,
                                     p.rope_cos.data_ptr(), p.rope_sin.data_ptr(), stream), "rope")
        _lib.check(lib.armt_attention(G, self.qkv.data_ptr(), 3 * d, T * 3 * d, self.ctx.data_ptr(), d, T * d,
                                      wout, T, cfg.n_heads, p.d_head, 1.0 / math.sqrt(p.d_head), stream),
                   "attention")

        def fill_o(a):
            a.M, a.N, a.K, a.ab_dtype = T, d, d, p.ab
            a.A, a.lda, a.a_stride = self.ctx.data_ptr(), d, T * d
            a.B, a.ldb, a.b_stride = p.wo.data_ptr(), d, d * d
            a.C, a.ldc, a.c_stride, a.c_dtype = self.xs.data_ptr(), d, T * d, F32
            a.epilogue = EPI_RESIDUAL
            a.R, a.ldr, a.r_stride = self.xs.data_ptr(), d, T * d
            if fused:
                a.C2, a.ldc2, a.c2_stride = self.xs_bf.data_ptr(), d, T * d
                a.ssq_out, a.ssq_stride, a.ssq_np = self.ssq_mlp.data_ptr(), T * self.ssq_np, self.ssq_np
            self._tables(a, gid, lrel, slots)
        _lib.check(lib.armt_gemm(self._gemm(("o",) + key, fill_o), stream), "o-proj")
        # MLP sub-block
        if not fused:
            _lib.check(lib.armt_rmsnorm(mem, self.xs.data_ptr(), T * d, p.unit_gain.data_ptr(), self.h.data_ptr(),
                                        wout, T * d, T, d, cfg.eps_norm, stream), "rmsnorm mlp")
        F = p.d_ff_pad

        def fill_gu(a):
            a.M, a.N, a.K, a.ab_dtype = T, 2 * F, d, p.ab
            a.A, a.lda, a.a_stride = a_in.data_ptr(), d, T * d
            a.B, a.ldb, a.b_stride = p.wgu.data_ptr(), d, 2 * F * d
            if self.bf16:
                a.C, a.ldc, a.c_stride, a.c_dtype = self.gu.data_ptr(), F, T * F, BF16
                a.epilogue = EPI_SWIGLU
                a.swiglu_block = p.swiglu_block
                if fused:
                    a.ssq_in, a.ssq_stride, a.ssq_np = self.ssq_mlp.data_ptr(), T * self.ssq_np, self.ssq_np
                    a.norm_d, a.norm_eps = d, cfg.eps_norm
            else:
                a.C, a.ldc, a.c_stride, a.c_dtype = self.gu_full.data_ptr(), 2 * F, T * 2 * F, F32
                a.epilogue = EPI_STORE
            self._tables(a, a_idx, lrel, gid)
        if self.probe is not None:
            self.probe(G, 0, stream)
        _lib.check(lib.armt_gemm(self._gemm(("gu",) + key, fill_gu), stream), "gate/up")
        if self.probe is not None:
            self.probe(G, 1, stream)
        if not self.bf16:
            _lib.check(lib.armt_swiglu(G, self.gu_full.data_ptr(), 2 * F, T * 2 * F, self.gu.data_ptr(), F, T * F,
                                       F32, T, F, p.swiglu_block, stream), "swiglu")

        def fill_down(a):
            a.M, a.N, a.K, a.ab_dtype = T, d, F, p.ab
            a.A, a.lda, a.a_stride = self.gu.data_ptr(), F, T * F
            a.B, a.ldb, a.b_stride = p.wdown.data_ptr(), F, d * F
            a.C, a.ldc, a.c_stride, a.c_dtype = self.xs.data_ptr(), d, T * d, F32
            a.epilogue = EPI_RESIDUAL
            a.R, a.ldr, a.r_stride = self.xs.data_ptr(), d, T * d
            if self.bf16:
                a.C2, a.ldc2, a.c2_stride = self.xs_bf.data_ptr(), d, T * d
            self._tables(a, gid, lrel, slots)
        _lib.check(lib.armt_gemm(self._gemm(("down",) + key, fill_down), stream), "down-proj")

    def update(self, slots, layers, state: MemoryState, stream: int, state_layers=None) -> None:
        """update_stack (armt/memory.py:155-180) from the memory rows of xs[slots]
        (``state_layers``: see ``retrieve``)."""
        if self.cfg.num_mem_tokens == 0:
            return
        self.project_kvb(slots, layers, stream)
        self.fold(slots, layers, state, stream, state_layers)

    def project_kvb(self, slots, layers, stream: int) -> None:
        """k, v, beta projections of the memory rows (armt/memory.py:166-171) into ``self.kvb``."""
        p, cfg, lib = self.p, self.cfg, self.lib
        T, d, M = p.T, cfg.d_model, cfg.num_mem_tokens
        lrel = [l - self.layer_base for l in layers]
        gid = list(range(len(layers)))
        src = self.xs_bf if self.bf16 else self.xs
        esz = src.element_size()

        def fill_kvb(a):
            a.M, a.N, a.K, a.ab_dtype = M, p.n_kvb, d, p.ab
            a.A, a.lda, a.a_stride = src.data_ptr() + cfg.segment_size * d * esz, d, T * d
            a.B, a.ldb, a.b_stride = p.wkvb.data_ptr(), d, p.n_kvb * d
            a.C, a.ldc, a.c_stride, a.c_dtype = self.kvb.data_ptr(), p.n_kvb, M * p.n_kvb, F32
            a.epilogue = EPI_STORE
            self._tables(a, slots, lrel, gid)
        _lib.check(lib.armt_gemm(self._gemm(("kvb", tuple(slots), tuple(layers)), fill_kvb), stream), "kvb")

    def fold(self, slots, layers, state: MemoryState, stream: int, state_layers=None) -> None:
        """The delta-rule fold of update_stack (armt/memory.py:94-125, 175-180) from
        the k/v/beta projections already in ``self.kvb``."""
        if state_layers is None:
            state_layers = layers
        p, cfg, lib = self.p, self.cfg, self.lib
        d, M = cfg.d_model, cfg.num_mem_tokens
        mem = self._members(slots, state_layers)
        if self.bf16:
            _lib.check(lib.armt_mem_fold_tc(mem, self.kvb.data_ptr(), p.n_kvb, M * p.n_kvb, p.v_off, p.k_off,
                                            p.b_off, state.A.data_ptr(), state.z.data_ptr(), state.memop.data_ptr(),
                                            d, M, cfg.d_mem, cfg.dpfp_nu, p.eps_assoc, self.fold_ws.data_ptr(),
                                            stream), "mem_fold_tc")
        else:
            _lib.check(lib.armt_mem_fold(mem, self.kvb.data_ptr(), p.n_kvb, M * p.n_kvb, p.v_off, p.k_off,
                                         p.b_off, state.A.data_ptr(), state.z.data_ptr(), None, 0, d, M,
                                         cfg.d_mem, cfg.dpfp_nu, p.eps_assoc, self.fold_ws.data_ptr(), stream),
                       "mem_fold")

    def step(self, slots, layers, state: MemoryState, stream: int, state_layers=None) -> None:
        self.retrieve(slots, layers, state, stream, state_layers)
        self.forward(slots, layers, stream)
        self.update(slots, layers, state, stream, state_layers)

    def _full_vocab(self) -> None:
        if self.p.unemb.shape[0] != self.cfg.vocab_size:
            raise InputError("these prepared weights hold one vocab block; use unembed_block")

    def unembed_lse(self, slot: int, ids: torch.Tensor, row0: int, n_tokens: int, part: torch.Tensor,
                    tgt: torch.Tensor, stream: int, max_ctas: int = 0) -> None:
        """LM head with the fused next-token NLL epilogue: no logits are written;
        per row and 256-wide vocab tile (max, sum exp) partials + the target logit."""
        p, cfg = self.p, self.cfg
        d, V, seg = cfg.d_model, cfg.vocab_size, cfg.segment_size
        src = self.xs_bf if self.bf16 else self.xs
        rows = max(0, min(seg, n_tokens - 1 - row0))
        tiles = part.shape[1]
        self._full_vocab()

        def fill(a):
            a.M, a.N, a.K, a.ab_dtype = seg, V, d, p.ab
            a.A, a.lda, a.a_stride = src.data_ptr(), d, p.T * d
            a.B, a.ldb, a.b_stride = p.unemb.data_ptr(), d, V * d
            a.C, a.ldc, a.c_stride, a.c_dtype = tgt.data_ptr(), 1, 0, F32  # unused by the LSE epilogue
            a.epilogue = _lib.EPI_LSE
            a.lse_part, a.lse_ld = part.data_ptr() + row0 * tiles * 8, tiles
            a.targets = ids.data_ptr() + (row0 + 1) * 8
            a.lse_tgt, a.lse_rows = tgt.data_ptr() + row0 * 4, rows
            a.max_ctas = max_ctas
            self._tables(a, [slot], [0], [0])
        _lib.check(self.lib.armt_gemm(self._gemm(("lse", slot, part.data_ptr(), row0, rows, max_ctas), fill), stream),
                   "unembed (fused nll)")

    def unembed(self, slot: int, out: torch.Tensor, row0: int, stream: int, max_ctas: int = 0) -> None:
        """armt/layers.py:321-323: logits rows [row0, row0+seg) = xs[slot][:seg] @ U."""
        p, cfg = self.p, self.cfg
        d, V, seg = cfg.d_model, cfg.vocab_size, cfg.segment_size
        src = self.xs_bf if self.bf16 else self.xs
        odt = BF16 if out.dtype == torch.bfloat16 else F32
        self._full_vocab()

        def fill(a):
            a.M, a.N, a.K, a.ab_dtype = seg, V, d, p.ab
            a.A, a.lda, a.a_stride = src.data_ptr(), d, p.T * d
            a.B, a.ldb, a.b_stride = p.unemb.data_ptr(), d, V * d
            a.C, a.ldc, a.c_stride, a.c_dtype = out.data_ptr() + row0 * V * out.element_size(), V, seg * V, odt
            a.epilogue = EPI_STORE
            a.max_ctas = max_ctas
            self._tables(a, [slot], [0], [0])
        _lib.check(self.lib.armt_gemm(self._gemm(("lm", slot, out.data_ptr(), row0, max_ctas), fill), stream),
                   "unembed")

    def unembed_block(self, a_ptr: int, a_ld: int, v0: int, v1: int, row0: int, stream: int,
                      out: torch.Tensor | None = None, lse=None, key=None) -> None:
        """LM head rows [row0, row0+seg) over the vocab block [v0, v1) (vocab-parallel
        head of the layer-sharded path): A = seg x d bf16 rows at ``a_ptr`` (leading
        dimension ``a_ld``). ``out`` = this rank's logits block (rows, v1-v0), or
        ``lse`` = (part, tgt, targets_local, n_tokens) for the fused next-token NLL
        partials (targets_local = ids - v0, so only this block's targets match)."""
        p, cfg = self.p, self.cfg
        d, V, seg = cfg.d_model, cfg.vocab_size, cfg.segment_size
        nv = v1 - v0

        def fill(a):
            a.M, a.N, a.K, a.ab_dtype = seg, nv, d, p.ab
            a.A, a.lda, a.a_stride = a_ptr, a_ld, seg * a_ld
            if not (p.vocab_base <= v0 <= v1 <= p.vocab_base + p.unemb.shape[0]):
                raise InputError(f"vocab block [{v0}, {v1}) not held by these weights "
                                 f"(columns {p.vocab_base}..{p.vocab_base + p.unemb.shape[0]})")
            a.B, a.ldb, a.b_stride = p.unemb.data_ptr() + (v0 - p.vocab_base) * d * p.unemb.element_size(), d, V * d
            if lse is None:
                odt = BF16 if out.dtype == torch.bfloat16 else F32
                a.C, a.ldc, a.c_stride, a.c_dtype = out.data_ptr() + row0 * nv * out.element_size(), nv, seg * nv, odt
                a.epilogue = EPI_STORE
            else:
                part, tgt, tloc, n_tokens = lse
                tiles = part.shape[1]
                rows = max(0, min(seg, n_tokens - 1 - row0))
                a.C, a.ldc, a.c_stride, a.c_dtype = tgt.data_ptr(), 1, 0, F32
                a.epilogue = _lib.EPI_LSE
                a.lse_part, a.lse_ld = part.data_ptr() + row0 * tiles * 8, tiles
                a.targets = tloc.data_ptr() + (row0 + 1) * 8
                a.lse_tgt, a.lse_rows = tgt.data_ptr() + row0 * 4, rows
            self._tables(a, [0], [0], [0])
        k = ("blk", a_ptr, v0, v1, row0, None if out is None else out.data_ptr(), lse is None) if key is None else key
        _lib.check(self.lib.armt_gemm(self._gemm(k, fill), stream), "unembed (vocab block)")
