"""CPU oracle for the ARMT segment-recurrent forward — TEST INFRASTRUCTURE.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it. The device path in
``paper_2506_05229_b200`` never routes through it and fails loudly when
its CUDA library is missing.

It restates, in NumPy, the algorithm of the reference package
(``/root/reference/pkg/src/armt``), function by function, citing the
reference file:line each one follows. It is pinned against golden vectors
produced by running the reference itself in the build container
(``scripts/make_golden.py`` → ``tests/golden/*.npz``; checked by
``tests/test_oracle.py``), so parity here is "pinned", not "unpinned".

Matrix products use BLAS (``@``) rather than the reference's strictly
ascending-k numba loops (armt/tensor_ops.py:31-45): in f64 that changes
results only at the 1e-15 level, which the tolerance tests absorb.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

ROPE_BASE = 10000.0  # armt/config.py:27


# ---------------------------------------------------------------------------
# configuration view (any object with the reference's ModelConfig fields)
# ---------------------------------------------------------------------------

def derived(cfg):
    """d_head, d_phi, T (armt/config.py:63-74)."""
    return cfg.d_model // cfg.n_heads, 2 * cfg.dpfp_nu * cfg.d_mem, cfg.segment_size + cfg.num_mem_tokens


# ---------------------------------------------------------------------------
# elementwise pieces
# ---------------------------------------------------------------------------

def dpfp(x: np.ndarray, nu: int) -> np.ndarray:
    """DPFP-nu feature map (armt/memory.py:34-45).

    r = [relu(x), relu(-x)]; block j (1..nu) is r * roll(r, -j), i.e.
    out[(j-1)*2m + i] = r[i] * r[(i + j) mod 2m].
    """
    r = np.concatenate([np.maximum(x, 0), np.maximum(-x, 0)], axis=-1)
    return np.concatenate([r * np.roll(r, -j, axis=-1) for j in range(1, nu + 1)], axis=-1)


def sigmoid(x: np.ndarray) -> np.ndarray:
    """Stable logistic (armt/layers.py:149-156)."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def rms_norm(x: np.ndarray, gain: np.ndarray, eps: float) -> np.ndarray:
    """x / sqrt(mean(x^2) + eps) * gain (armt/tensor_ops.py:267-281)."""
    ms = np.mean(x * x, axis=-1, keepdims=True)
    return x / np.sqrt(ms + eps) * gain


def rope_tables(T: int, d_head: int, dtype=np.float64):
    """cos/sin over positions 0..T-1, restarting every segment
    (armt/layers.py:101-106, 131-132)."""
    inv = ROPE_BASE ** (-np.arange(0, d_head, 2, dtype=np.float64) / d_head)
    ang = np.arange(T, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(dtype), np.sin(ang).astype(dtype)


def apply_rope(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Rotate-half RoPE on (..., T, d_head) (armt/layers.py:169-176)."""
    h = cos.shape[1]
    a, b = x[..., :h], x[..., h:]
    return np.concatenate([a * cos - b * sin, b * cos + a * sin], axis=-1)


# ---------------------------------------------------------------------------
# one (segment, layer) cell: retrieve -> block -> update
# ---------------------------------------------------------------------------

@dataclass
class LayerWeights:
    """One layer's slice, reference layouts (armt/weights.py:27-50)."""
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w_gate: np.ndarray
    w_in: np.ndarray
    w_out: np.ndarray
    attn_gain: np.ndarray
    mlp_gain: np.ndarray
    w_k_mem: np.ndarray
    w_v_mem: np.ndarray
    w_beta: np.ndarray
    w_q_assoc: np.ndarray


def layer_slice(weights, l: int, dtype) -> LayerWeights:
    g = lambda name: np.asarray(getattr(weights, name)[l], dtype=dtype)
    return LayerWeights(*(g(n) for n in ("wq", "wk", "wv", "wo", "w_gate", "w_in", "w_out",
                                         "attn_gain", "mlp_gain", "w_k_mem", "w_v_mem",
                                         "w_beta", "w_q_assoc")))


def retrieve(A: np.ndarray, z: np.ndarray, x: np.ndarray, w_q_assoc: np.ndarray,
             nu: int, eps: float) -> np.ndarray:
    """Guarded associative readout added to the residual (armt/memory.py:132-152).

    q = x W_qa^T; phi = DPFP(q); x + (|phi.z| <= eps ? 0 : (phi A^T)/(phi.z)).
    """
    phi = dpfp(x @ w_q_assoc.T, nu)
    num = phi @ A.T
    den = phi @ z
    guarded = np.abs(den) <= eps
    safe = np.where(guarded, 1.0, den)
    return x + np.where(guarded[:, None], 0.0, num / safe[:, None])


def block(x: np.ndarray, lw: LayerWeights, n_heads: int, eps_norm: float,
          cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Pre-norm LLaMA-style block (armt/layers.py:197-246).

    MHA with rotate-half RoPE and an additive causal mask over all T rows
    (memory rows last), then SwiGLU MLP; both sub-blocks residual.
    """
    T, d = x.shape
    dh = d // n_heads
    h = rms_norm(x, lw.attn_gain, eps_norm)
    split = lambda a: a.reshape(T, n_heads, dh).transpose(1, 0, 2)
    q = apply_rope(split(h @ lw.wq), cos, sin)
    k = apply_rope(split(h @ lw.wk), cos, sin)
    v = split(h @ lw.wv)
    scores = (q @ k.transpose(0, 2, 1)) * (1.0 / math.sqrt(dh))
    scores = scores + np.where(np.triu(np.ones((T, T), bool), 1), -np.inf, 0.0)
    scores = np.exp(scores - scores.max(-1, keepdims=True))
    probs = scores / scores.sum(-1, keepdims=True)
    ctx = (probs @ v).transpose(1, 0, 2).reshape(T, d)
    x = x + ctx @ lw.wo
    h = rms_norm(x, lw.mlp_gain, eps_norm)
    gate = h @ lw.w_gate
    return x + ((gate * sigmoid(gate)) * (h @ lw.w_in)) @ lw.w_out


def fold(A: np.ndarray, z: np.ndarray, m: np.ndarray, lw: LayerWeights, nu: int,
         eps: float, log: list | None = None) -> None:
    """Delta-rule write of M memory-token outputs, in token order, in place
    (armt/memory.py:155-180 projections, armt/memory.py:94-125 fold).

    For token i: zq = z.phi_i, nrm = phi_i.phi_i;
    vbar = |zq| <= eps ? 0 : (A phi_i)/zq; gamma = nrm <= eps ? 0 : 1 - zq/nrm;
    A += beta_i (v_i - vbar) phi_i^T; z += gamma phi_i.
    ``log`` (test diagnostics) receives (zq, nrm) for every token.
    """
    k = m @ lw.w_k_mem.T
    v = m @ lw.w_v_mem.T
    beta = sigmoid((m @ lw.w_beta.T)[:, 0])
    phi = dpfp(k, nu)
    for i in range(m.shape[0]):
        p = phi[i]
        zq = float(z @ p)
        nrm = float(p @ p)
        if log is not None:
            log.append((zq, nrm))
        vbar = np.zeros(A.shape[0], A.dtype) if abs(zq) <= eps else (A @ p) / zq
        gamma = 0.0 if nrm <= eps else 1.0 - zq / nrm
        A += np.outer(beta[i] * (v[i] - vbar), p)
        z += gamma * p


# ---------------------------------------------------------------------------
# executors
# ---------------------------------------------------------------------------

@dataclass
class OracleState:
    """MemoryState (armt/memory.py:52-87): A (L,d,d_phi), z (L,d_phi), updates (L,)."""
    A: np.ndarray
    z: np.ndarray
    updates: np.ndarray

    @classmethod
    def fresh(cls, cfg, dtype=np.float64):
        _, dphi, _ = derived(cfg)
        L, d = cfg.n_layers, cfg.d_model
        return cls(np.zeros((L, d, dphi), dtype), np.zeros((L, dphi), dtype), np.zeros(L, np.int64))


def segment_input(tokens, cfg):
    """Pad the tail segment with id 0 (armt/executors.py:74-92)."""
    ids = np.asarray(tokens, dtype=np.int64)
    n = ids.shape[0]
    pad = (-n) % cfg.segment_size
    if pad:
        ids = np.concatenate([ids, np.zeros(pad, np.int64)])
    return ids.reshape(-1, cfg.segment_size), n


class Oracle:
    """Reference forward in one precision over host weights."""

    def __init__(self, weights, cfg, dtype=np.float64, eps_assoc: float | None = None):
        self.cfg = cfg
        self.dtype = np.dtype(dtype)
        self.dh, self.dphi, self.T = derived(cfg)
        if eps_assoc is None:
            eps_assoc = cfg.eps_assoc if cfg.eps_assoc is not None else (
                1e-12 if self.dtype == np.float64 else 1e-6)
        self.eps = float(eps_assoc)
        self.layers = [layer_slice(weights, l, self.dtype) for l in range(cfg.n_layers)]
        self.embedding = np.asarray(weights.embedding, self.dtype)
        self.mem_embedding = np.asarray(weights.mem_embedding, self.dtype)
        self.unembedding = np.asarray(weights.unembedding, self.dtype)
        self.cos, self.sin = rope_tables(self.T, self.dh, self.dtype)
        self.fold_log = None   # set to a list to record (layer, [(zq, nrm) per token]) per fold

    def embed(self, ids):
        """armt/layers.py:306-318."""
        return np.concatenate([self.embedding[ids], self.mem_embedding])

    def cell(self, state: OracleState, l: int, x: np.ndarray) -> np.ndarray:
        """retrieve -> block -> update for node (s, l) (armt/executors.py:137-143)."""
        cfg = self.cfg
        lw = self.layers[l]
        x = retrieve(state.A[l], state.z[l], x, lw.w_q_assoc, cfg.dpfp_nu, self.eps)
        y = block(x, lw, cfg.n_heads, cfg.eps_norm, self.cos, self.sin)
        rows = [] if self.fold_log is not None else None
        fold(state.A[l], state.z[l], y[cfg.segment_size:], lw, cfg.dpfp_nu, self.eps, rows)
        if rows is not None:
            self.fold_log.append((l, rows))
        state.updates[l] += 1
        return y

    def unembed(self, y):
        """Token rows only, no final norm (armt/layers.py:321-323)."""
        return y[:self.cfg.segment_size] @ self.unembedding

    def run_sequential(self, tokens, state: OracleState | None = None):
        """armt/executors.py:123-150: segments outer, layers inner."""
        segs, n = segment_input(tokens, self.cfg)
        state = state or OracleState.fresh(self.cfg, self.dtype)
        rows, nodes = [], []
        for s, ids in enumerate(segs):
            x = self.embed(ids)
            for l in range(self.cfg.n_layers):
                x = self.cell(state, l, x)
                nodes.append([(s, l)])
            rows.append(self.unembed(x))
        return np.concatenate(rows)[:n], state, nodes

    def run_diagonal(self, tokens, state: OracleState | None = None):
        """armt/executors.py:153-226: anti-diagonal wavefront; members in
        ascending layer order; exiting segments unembedded."""
        segs, n = segment_input(tokens, self.cfg)
        S, L = len(segs), self.cfg.n_layers
        state = state or OracleState.fresh(self.cfg, self.dtype)
        flying: list[list] = []   # [segment, layer_cursor, activation]
        rows = [None] * S
        nodes = []
        nxt = 0
        while nxt < S or flying:
            if nxt < S:
                flying.insert(0, [nxt, 0, self.embed(segs[nxt])])
                nxt += 1
            nodes.append([(m[0], m[1]) for m in flying])
            for m in flying:
                m[2] = self.cell(state, m[1], m[2])
                m[1] += 1
            done = [m for m in flying if m[1] == L]
            for m in done:
                rows[m[0]] = self.unembed(m[2])
            flying = [m for m in flying if m[1] < L]
        return np.concatenate(rows)[:n], state, nodes


def relative_error(a, b) -> float:
    """||a-b||_F / ||b||_F in f64; 0 if both zero (armt/executors.py:233-247)."""
    a64 = np.asarray(a, np.float64)
    b64 = np.asarray(b, np.float64)
    base = float(np.linalg.norm(b64))
    diff = float(np.linalg.norm(a64 - b64))
    if base == 0.0:
        return 0.0 if diff == 0.0 else float("inf")
    return diff / base


def time_cells(oracle: Oracle, n_cells: int, seed: int = 0) -> float:
    """Seconds per full-width (segment, layer) cell, measured on this host
    (the CPU-baseline sample used by bench.py)."""
    rng = np.random.default_rng(seed)
    state = OracleState.fresh(oracle.cfg, oracle.dtype)
    x = oracle.embed(rng.integers(0, oracle.cfg.vocab_size, oracle.cfg.segment_size))
    t0 = time.perf_counter()
    for c in range(n_cells):
        x = oracle.cell(state, c % oracle.cfg.n_layers, x)
    return (time.perf_counter() - t0) / n_cells
