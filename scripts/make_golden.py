"""Generate golden vectors by running the REFERENCE package in this container.

Run (build container only; /root/reference does not exist on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python scripts/make_golden.py

Outputs small ``.npz`` fixtures under ``tests/golden/``. They pin the
NumPy oracle (``tests/test_oracle.py``) and the device path
(``tests/test_gpu_*.py``) to the reference's own outputs.

Fixtures
--------
small_ref   reference test fixture (``pkg/tests/conftest.py:39-48``): L=3,
            d=16, damped w_v_mem, default eps, f64; 3 segments.
c1_cond     BASELINE config C1, conditioned per SURVEY
            Appendix B (eps_assoc=1.0, w_v_mem x 1/32) with every weight
            rounded onto the bf16 grid, 8 segments, f64 and f32 runs.
mid_cond    d=256, L=4, 4 heads (d_head 64), seg 128, M 16, d_mem 16,
            eps_assoc 10 (Appendix B row), bf16-grid weights, 6 segments.
ops_c1      per-core goldens on C1: retrieve_stack / forward_stack /
            update_stack on a live memory state (after 2 segments), G=2.
traces      reference node lists of run_diagonal for (S, L) grids.
"""

from __future__ import annotations

import hashlib
import os
import sys
from dataclasses import replace

import numpy as np

import armt
from armt import ModelConfig, init_weights, run_diagonal, run_sequential
from armt.layers import forward_stack, prepare_weights
from armt.memory import MemoryState, retrieve_stack, update_stack

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")
sys.path.insert(0, os.path.join(HERE, ".."))
from paper_2506_05229_b200.weights import round_to_bf16  # noqa: E402

C1 = dict(n_layers=2, d_model=128, n_heads=4, d_ff=512, segment_size=64,
          num_mem_tokens=16, d_mem=16, vocab_size=256)
MID = dict(n_layers=4, d_model=256, n_heads=4, d_ff=512, segment_size=128,
           num_mem_tokens=16, d_mem=16, vocab_size=512)


def cli_tokens(cfg, n, seed=0):
    """armt/cli.py:45-49 token convention."""
    return np.random.default_rng([seed, n]).integers(0, cfg.vocab_size, n, dtype=np.int64)


def conditioned(cfg, damp=1.0 / 32):
    w = init_weights(cfg)
    w = replace(w, w_v_mem=w.w_v_mem * damp)
    fields = {k: round_to_bf16(v) for k, v in w.__dict__.items() if isinstance(v, np.ndarray)}
    return replace(w, **fields)


def weight_digest(w):
    h = hashlib.sha256()
    for name in ("embedding", "mem_embedding", "wq", "wk", "wv", "wo", "w_gate", "w_in",
                 "w_out", "attn_gain", "mlp_gain", "w_k_mem", "w_v_mem", "w_beta",
                 "w_q_assoc", "unembedding"):
        h.update(np.ascontiguousarray(getattr(w, name), np.float64).tobytes())
    return h.hexdigest()


def run_both(w, cfg, tokens, dtype):
    st_s = MemoryState.fresh(cfg, dtype)
    st_d = MemoryState.fresh(cfg, dtype)
    seq, tr_s = run_sequential(w, cfg, tokens, dtype=dtype, state=st_s)
    diag, tr_d = run_diagonal(w, cfg, tokens, dtype=dtype, state=st_d)
    assert np.array_equal(seq, diag), "reference schedules disagree"
    nodes = [[[n.segment, n.layer] for n in ev.nodes] for ev in tr_d.events]
    return seq, st_s, nodes


def _trace_cfg(L):
    return ModelConfig(n_layers=L, d_model=8, n_heads=2, d_ff=8, segment_size=2,
                       num_mem_tokens=1, d_mem=1, vocab_size=7, seed=1)


def make_traces():
    """Reference node lists of run_diagonal (plain and under shuffle_seed, the
    reference's member-order audit hook, armt/executors.py:192-195) and of
    run_sequential, for several (S, L) grids."""
    grids = [(4, 3), (3, 2), (1, 5), (5, 1), (7, 4)]
    tr = {}
    for S, L in grids:
        cfg = _trace_cfg(L)
        toks = np.arange(S * 2) % 7
        _, trace = run_diagonal(init_weights(cfg), cfg, toks)
        flat = [[n.segment, n.layer] for ev in trace.events for n in ev.nodes]
        tr[f"nodes_{S}x{L}"] = np.array(flat, np.int64)
        tr[f"counts_{S}x{L}"] = np.array([len(ev.nodes) for ev in trace.events], np.int64)
    for S, L, seed in [(4, 3, 7), (7, 4, 123), (9, 6, 2024), (16, 16, 5)]:
        cfg = _trace_cfg(L)
        toks = np.arange(S * 2) % 7
        _, trace = run_diagonal(init_weights(cfg), cfg, toks, shuffle_seed=seed)
        flat = [[n.segment, n.layer] for ev in trace.events for n in ev.nodes]
        tr[f"shuf_nodes_{S}x{L}_seed{seed}"] = np.array(flat, np.int64)
        tr[f"shuf_counts_{S}x{L}_seed{seed}"] = np.array([len(ev.nodes) for ev in trace.events], np.int64)
    for S, L in [(3, 4)]:
        cfg = _trace_cfg(L)
        _, trace = run_sequential(init_weights(cfg), cfg, np.arange(S * 2) % 7)
        tr[f"seq_nodes_{S}x{L}"] = np.array([[n.segment, n.layer] for ev in trace.events for n in ev.nodes],
                                            np.int64)
    np.savez_compressed(os.path.join(OUT, "traces.npz"), **tr)


def make_containers():
    """Weight containers written by the reference's own save_weights
    (armt/weights.py:145-171): the reference's test config (tests/test_container.py:12-16)
    in f64 and f32 payloads, and a C1-shaped f32 container that the GPU loader test runs."""
    from armt import save_weights
    cfg = ModelConfig(n_layers=2, d_model=8, n_heads=2, d_ff=12, segment_size=3,
                      num_mem_tokens=2, d_mem=3, vocab_size=17, seed=5)
    w = init_weights(cfg)
    save_weights(w, os.path.join(OUT, "ref_tiny_f64.armt"))
    w32 = replace(w, **{k: v.astype(np.float32) for k, v in w.named_arrays().items()})
    save_weights(w32, os.path.join(OUT, "ref_tiny_f32.armt"))
    cfg = ModelConfig(**C1, eps_assoc=1.0, seed=0)
    wc = conditioned(cfg)
    wc = replace(wc, **{k: v.astype(np.float32) for k, v in wc.named_arrays().items()})
    save_weights(wc, os.path.join(OUT, "ref_c1_cond_f32.armt"))


def main():
    os.makedirs(OUT, exist_ok=True)
    print("reference armt", armt.__version__)
    if len(sys.argv) > 1:   # e.g. `make_golden.py traces containers`: regenerate only those
        for name in sys.argv[1:]:
            globals()["make_" + name]()
        return

    # -- small_ref: the reference's own fixture ----------------------------
    cfg = ModelConfig(n_layers=3, d_model=16, n_heads=2, d_ff=32, segment_size=6,
                      num_mem_tokens=2, d_mem=4, vocab_size=50, seed=7)
    raw = init_weights(cfg)
    w = replace(raw, w_v_mem=raw.w_v_mem * 0.03125)
    tokens = np.random.default_rng(3).integers(0, cfg.vocab_size, 3 * cfg.segment_size,
                                               dtype=np.int64)
    logits, st, nodes = run_both(w, cfg, tokens, "f64")
    np.savez_compressed(os.path.join(OUT, "small_ref.npz"), tokens=tokens, logits=logits,
                        A=st.A, z=st.z, updates=st.updates,
                        digest=np.array(weight_digest(raw)))

    # -- c1_cond ------------------------------------------------------------
    cfg = ModelConfig(**C1, eps_assoc=1.0, seed=0)
    w = conditioned(cfg)
    n = 8 * cfg.segment_size
    tokens = cli_tokens(cfg, n)
    out = dict(tokens=tokens, digest=np.array(weight_digest(init_weights(cfg))))
    for dt in ("f64", "f32"):
        logits, st, nodes = run_both(w, cfg, tokens, dt)
        out[f"logits_{dt}"] = logits.astype(np.float32)
        out[f"A_{dt}"] = st.A.astype(np.float32)
        out[f"z_{dt}"] = st.z.astype(np.float32)
        out[f"updates_{dt}"] = st.updates
    # memory liveness: logits with inert memory (w_k_mem = 0, w_q_assoc kept)
    inert = replace(w, w_k_mem=np.zeros_like(w.w_k_mem))
    out["logits_inert_f64"] = run_sequential(inert, cfg, tokens, dtype="f64")[0].astype(np.float32)
    out["nodes"] = np.array([x for step in nodes for x in step], np.int64)
    out["node_counts"] = np.array([len(s) for s in nodes], np.int64)
    np.savez_compressed(os.path.join(OUT, "c1_cond.npz"), **out)

    # -- mid_cond -------------------------------------------------------------
    cfg = ModelConfig(**MID, eps_assoc=10.0, seed=0)
    w = conditioned(cfg)
    n = 6 * cfg.segment_size - 37          # ragged tail: exercises padding
    tokens = cli_tokens(cfg, n)
    logits, st, _ = run_both(w, cfg, tokens, "f64")
    np.savez_compressed(os.path.join(OUT, "mid_cond.npz"), tokens=tokens,
                        logits=logits.astype(np.float32), A=st.A.astype(np.float32),
                        z=st.z.astype(np.float32), updates=st.updates)

    # -- ops_c1: per-core goldens on a live state ---------------------------
    cfg = ModelConfig(**C1, eps_assoc=1.0, seed=0)
    w = conditioned(cfg)
    tokens = cli_tokens(cfg, 2 * cfg.segment_size)
    out = {}
    for dt in ("f64", "f32"):
        st = MemoryState.fresh(cfg, dt)
        run_sequential(w, cfg, tokens, dtype=dt, state=st)
        prepared = prepare_weights(w, dt)
        rng = np.random.default_rng(5)
        x = rng.standard_normal((2, cfg.tokens_per_segment, cfg.d_model)).astype(prepared.dtype)
        layers = np.array([0, 1], np.int64)
        A0, z0 = st.A.copy(), st.z.copy()
        xr = retrieve_stack(st, layers, x, prepared)
        y = forward_stack(prepared, layers, x)
        update_stack(st, layers, y[:, -cfg.num_mem_tokens:, :], prepared)
        out.update({f"A0_{dt}": A0, f"z0_{dt}": z0, f"x_{dt}": x, f"retrieved_{dt}": xr,
                    f"forward_{dt}": y, f"A1_{dt}": st.A, f"z1_{dt}": st.z})
    np.savez_compressed(os.path.join(OUT, "ops_c1.npz"), **out)

    make_traces()
    make_containers()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
