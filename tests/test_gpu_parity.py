"""End-to-end parity of the device path with the reference (``-m gpu``).

Goldens come from running the reference package itself
(scripts/make_golden.py); the oracle (oracle/armt_oracle.py) is used for
configurations without a stored golden. Tolerances (relative Frobenius error,
the reference's own metric, armt/executors.py:233-247):

  * f32 mode  : 1e-4 on logits and on the final memory state (north star).
  * bf16 mode : 2e-2 on logits, 2e-2 on the final memory state, with the
    weights on the bf16 grid so both sides see identical weights; the error
    that remains is activation rounding, which grows with the number of
    segments, so it is asserted at the stated horizons.
  * schedule equivalence on the device: sequential == diagonal BITWISE, and
    shuffled member order == unshuffled BITWISE (lane-independent kernels).
"""

from dataclasses import replace

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import armt_oracle as O  # noqa: E402
from conftest import C1, MID, SMALL, golden  # noqa: E402
from fixtures import cli_tokens, conditioned_weights  # noqa: E402
import paper_2506_05229_b200 as P  # noqa: E402
from paper_2506_05229_b200.config import ModelConfig  # noqa: E402
from paper_2506_05229_b200.engine import MemoryState, prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import relative_error, run_diagonal, run_sequential  # noqa: E402

TOL = {"f32": 1e-4, "bf16": 2e-2}


@pytest.fixture(scope="module")
def c1():
    cfg = ModelConfig(**C1, eps_assoc=1.0)
    w = conditioned_weights(cfg)
    return cfg, w, {dt: prepare_weights(w, dt) for dt in ("f32", "bf16")}


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c1_logits_and_state_match_reference(c1, dtype):
    """Logits of all 8 segments within the mode's tolerance of the reference's
    f64 golden. The final memory state is held to the same tolerance in f32,
    and in bf16 whenever no fold of the oracle run sits near a high-gain guard
    boundary (GUARD_BAND below). The golden sequence has one: segment 4, layer
    0, |zq| within 15.5% of eps with nrm/|zq| = 6.4. There the bf16 state is
    held to the tolerance over the prefix BEFORE that fold
    (test_c1_state_before_first_guard_critical_fold) and to 0.25 at the end —
    over 12 token seeds the final bf16 A/z error has median 5e-3/6e-3 and
    outliers up to 0.12/0.08, where one seed's rounding noise lands a guard
    token on the other branch (scripts/c1_seed_spread.py, profiles/r2_parity.md)."""
    cfg, w, prep = c1
    g = golden("c1_cond")
    state = MemoryState.fresh(cfg)
    logits, trace = run_diagonal(prep[dtype], cfg, g["tokens"], dtype=dtype, state=state)
    A, z, upd = state.to_numpy()
    assert np.isfinite(logits).all()
    assert relative_error(logits, g["logits_f64"]) < TOL[dtype]
    critical = _c1_guard_critical_folds(cfg, w, g["tokens"]) if dtype == "bf16" else []
    tol_state = 0.25 if critical else TOL[dtype]
    assert relative_error(A, g["A_f64"]) < tol_state, critical
    assert relative_error(z, g["z_f64"]) < tol_state, critical
    assert np.array_equal(upd, g["updates_f64"])
    flat = np.array([[n.segment, n.layer] for ev in trace.events for n in ev.nodes])
    assert np.array_equal(flat, g["nodes"])


def _c1_guard_critical_folds(cfg, w, tokens):
    """(segment, layer) of every fold of the f64 oracle run with a token near a
    high-gain guard boundary, in execution order."""
    orc = O.Oracle(w, cfg, np.float64)
    orc.fold_log = []
    _, _, nodes = orc.run_diagonal(tokens)
    cells = [cell for step in nodes for cell in step]
    return [cells[i] for i, (layer, rows) in enumerate(orc.fold_log)
            if _guard_critical(rows, cfg.eps_assoc)]


def test_c1_state_before_first_guard_critical_fold(c1):
    """bf16 memory state held to 2e-2 over the longest prefix of the golden
    sequence whose folds all stay clear of a high-gain guard boundary."""
    cfg, w, prep = c1
    tokens = golden("c1_cond")["tokens"]
    critical = _c1_guard_critical_folds(cfg, w, tokens)
    n_seg = min([s for s, _ in critical], default=len(tokens) // cfg.segment_size)
    assert n_seg >= 3, critical
    prefix = tokens[:n_seg * cfg.segment_size]
    want, ostate, _ = O.Oracle(w, cfg, np.float64).run_diagonal(prefix)
    st = MemoryState.fresh(cfg)
    got, _ = run_diagonal(prep["bf16"], cfg, prefix, state=st)
    A, z, _ = st.to_numpy()
    assert relative_error(got, want) < TOL["bf16"]
    assert relative_error(A, ostate.A) < TOL["bf16"], (n_seg, relative_error(A, ostate.A))
    assert relative_error(z, ostate.z) < TOL["bf16"], (n_seg, relative_error(z, ostate.z))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_device_schedules_agree_bitwise(c1, dtype):
    cfg, _, prep = c1
    tokens = cli_tokens(cfg, 5 * cfg.segment_size, seed=3)
    s1, s2 = MemoryState.fresh(cfg), MemoryState.fresh(cfg)
    seq, _ = run_sequential(prep[dtype], cfg, tokens, dtype=dtype, state=s1)
    diag, _ = run_diagonal(prep[dtype], cfg, tokens, dtype=dtype, state=s2)
    assert np.array_equal(seq, diag)
    assert torch.equal(s1.A, s2.A) and torch.equal(s1.z, s2.z)


def test_mid_width_runs_are_deterministic_and_schedule_invariant():
    # d=256 spans several N tiles per row: exercises the fused-RMSNorm partial
    # sums (fixed-order, no atomics) for bitwise reproducibility
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    prep = prepare_weights(conditioned_weights(cfg), "bf16")
    tokens = cli_tokens(cfg, 5 * cfg.segment_size, seed=8)
    a, _ = run_diagonal(prep, cfg, tokens)
    b, _ = run_diagonal(prep, cfg, tokens)
    c, _ = run_sequential(prep, cfg, tokens)
    assert np.array_equal(a, b)
    assert np.array_equal(a, c)


def test_shuffle_and_graph_do_not_change_logits(c1):
    cfg, _, prep = c1
    tokens = cli_tokens(cfg, 6 * cfg.segment_size, seed=4)
    base, _ = run_diagonal(prep["bf16"], cfg, tokens)
    shuf, tr = run_diagonal(prep["bf16"], cfg, tokens, shuffle_seed=123)
    graphed, _ = run_diagonal(prep["bf16"], cfg, tokens, graph=True)
    assert np.array_equal(base, shuf)
    assert np.array_equal(base, graphed)


def test_state_carries_across_calls(c1):
    cfg, _, prep = c1
    tokens = cli_tokens(cfg, 4 * cfg.segment_size, seed=5)
    whole, _ = run_sequential(prep["bf16"], cfg, tokens)
    st = MemoryState.fresh(cfg)
    half = len(tokens) // 2
    a, _ = run_diagonal(prep["bf16"], cfg, tokens[:half], state=st)
    b, _ = run_diagonal(prep["bf16"], cfg, tokens[half:], state=st)
    assert np.array_equal(whole, np.concatenate([a, b]))
    assert st.updates.tolist() == [4] * cfg.n_layers


def test_inert_memory_restarts_rope_per_segment(c1):
    # pkg/tests/test_executors.py:111-120 on the device
    cfg, w, _ = c1
    inert = replace(w, w_k_mem=np.zeros_like(w.w_k_mem))
    prep = prepare_weights(inert, "bf16")
    seg = cli_tokens(cfg, cfg.segment_size, seed=6)
    logits, _ = run_sequential(prep, cfg, np.tile(seg, 2))
    S = cfg.segment_size
    assert np.array_equal(logits[:S], logits[S:])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_mid_ragged_tail_matches_reference(dtype):
    g = golden("mid_cond")
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    w = conditioned_weights(cfg)
    state = MemoryState.fresh(cfg)
    logits, _ = run_diagonal(w, cfg, g["tokens"], dtype=dtype, state=state)
    assert logits.shape == g["logits"].shape
    assert relative_error(logits, g["logits"]) < TOL[dtype]
    assert relative_error(state.A.cpu().numpy(), g["A"]) < TOL[dtype]


def test_reference_small_fixture_f32():
    # the reference's own test fixture (pkg/tests/conftest.py), default eps
    g = golden("small_ref")
    cfg = ModelConfig(**SMALL)
    raw = P.init_weights(cfg)
    w = replace(raw, w_v_mem=raw.w_v_mem * 0.03125)
    logits, _ = run_diagonal(w, cfg, g["tokens"], dtype="f32")
    assert relative_error(logits, g["logits"]) < 1e-4


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_per_core_ops_match_reference(c1, dtype):
    from paper_2506_05229_b200.layers import forward_stack, retrieve_stack, update_stack
    cfg, _, prep = c1
    g = golden("ops_c1")
    st = MemoryState.from_numpy(g["A0_f64"], g["z0_f64"], [2, 2])
    x = torch.tensor(g["x_f64"], dtype=torch.float32, device="cuda")
    xr = retrieve_stack(st, [0, 1], x, prep[dtype])
    assert relative_error(xr, g["retrieved_f64"]) < TOL[dtype]
    y = forward_stack(prep[dtype], [0, 1], x)
    assert relative_error(y, g["forward_f64"]) < TOL[dtype]
    update_stack(st, [0, 1], y[:, cfg.segment_size:].contiguous(), prep[dtype])
    assert relative_error(st.A.cpu().numpy(), g["A1_f64"]) < TOL[dtype]
    assert relative_error(st.z.cpu().numpy(), g["z1_f64"]) < TOL[dtype]


def kv_weights(cfg):
    # pkg/tests/test_memory.py:68-82: projections exposing key/value slots
    base = P.init_weights(cfg)
    L, dm = cfg.n_layers, cfg.d_model
    w_k = np.zeros((L, 1, dm)); w_k[:, 0, 7] = 1.0
    w_v = np.tile(np.eye(dm), (L, 1, 1)); w_v[:, 6:, :] = 0.0
    w_b = np.zeros((L, 1, dm)); w_b[:, 0, 6] = 50.0
    return replace(base, w_k_mem=w_k, w_v_mem=w_v, w_beta=w_b, w_q_assoc=w_k.copy())


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("key", [1.0, -1.0, 4.0, 0.0625])
def test_store_then_retrieve_is_exact(dtype, key):
    # pkg/tests/test_memory.py:99-113: power-of-two keys make every quotient exact
    from paper_2506_05229_b200.layers import SegmentActivation, assoc_retrieve, assoc_update
    cfg = ModelConfig(n_layers=2, d_model=8, n_heads=2, d_ff=8, segment_size=2, num_mem_tokens=1,
                      d_mem=1, vocab_size=9, seed=0)
    prep = prepare_weights(kv_weights(cfg), dtype)
    st = MemoryState.fresh(cfg)
    values = np.array([1.25, 1.5, 1.9921875, 1.0, 1.75], np.float32)
    row = np.zeros((1, 8), np.float32); row[0, :5] = values; row[0, 6] = 1.0; row[0, 7] = key
    assoc_update(st, 0, torch.tensor(row, device="cuda"), prep)
    assert st.updates.tolist() == [1, 0]
    q = np.zeros((cfg.tokens_per_segment, 8), np.float32); q[:, 7] = key
    act = SegmentActivation(torch.tensor(q, device="cuda"), 2, 0)
    out = assoc_retrieve(st, 0, act, prep).data.cpu().numpy()
    assert np.array_equal(out[0, :5], values)
    out1 = assoc_retrieve(st, 1, act, prep).data.cpu().numpy()
    assert np.array_equal(out1[0, :5], np.zeros(5, np.float32))


def test_fused_scoring_nll_matches_logits_path():
    # LM-head epilogue NLL (no logits materialised) vs log-softmax of the logits
    from paper_2506_05229_b200.executors import Session
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    prep = prepare_weights(conditioned_weights(cfg), "bf16")
    n = 4 * cfg.segment_size - 5
    tokens = torch.as_tensor(cli_tokens(cfg, n, seed=9)).cuda()
    plain = Session(prep, n, graph=False)
    logits = plain.forward(tokens).float()
    want = -torch.log_softmax(logits[:-1].double(), -1).gather(1, tokens[1:, None])[:, 0]
    via_kernel = plain.nll(tokens)
    scoring = Session(prep, n, scoring=True)
    got = scoring.nll(tokens)
    assert scoring.runner.logits is None
    assert float((via_kernel.double() - want).abs().max()) < 1e-3
    # the fused path works from fp32 accumulators, the reference side from bf16-rounded
    # logits (|logit| ~ 10 -> ~0.04 rounding): bound that difference, not equality
    diff = (got.double() - want).abs()
    assert float(diff.max()) < 0.05 and float(diff.mean()) < 5e-3
    assert abs(float(got.double().mean() - want.mean())) < 2e-3


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_minibatch_copies_equal_sequential_bitwise(c1, dtype):
    """Minibatch mode (armt/cli.py:139-153): every copy of the lockstep grouped
    run reproduces the one-stream sequential run bitwise, state blocks included."""
    from paper_2506_05229_b200.executors import run_minibatch
    cfg, _, prep = c1
    tokens = cli_tokens(cfg, 4 * cfg.segment_size - 5, seed=9)
    ref_state = MemoryState.fresh(cfg)
    want, _ = run_sequential(prep[dtype], cfg, tokens, dtype=dtype, state=ref_state)
    copies = 3
    st = MemoryState.fresh(cfg, n_layers=copies * cfg.n_layers)
    got, trace = run_minibatch(prep[dtype], cfg, tokens, copies, dtype=dtype, state=st)
    assert got.shape == (copies,) + want.shape
    for b in range(copies):
        assert np.array_equal(got[b], want)
        L = cfg.n_layers
        assert torch.equal(st.A[b * L:(b + 1) * L], ref_state.A)
    assert trace.steps_executed == 4 * cfg.n_layers


def test_full_width_c2_layers_match_oracle():
    """C2 layer shapes at full width (d 2048, 32 heads of 64, d_ff 8192, segment
    1024 + 128 memory tokens, d_mem 64) through the real kernel paths (CTA-pair
    / multicast GEMMs, concurrent remainder, fused DPFP, ping-pong attention,
    tensor-core fold), 2 layers x 3 segments, against the f32 oracle. The vocab
    is cut to 4096 to keep the CPU oracle to seconds; tolerances as in the
    small configs (bf16 2e-2, f32 mode 1e-4)."""
    cfg = ModelConfig(n_layers=2, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024, num_mem_tokens=128,
                      d_mem=64, vocab_size=4096, eps_assoc=100.0, seed=0)
    w = conditioned_weights(cfg)
    tokens = cli_tokens(cfg, 3 * cfg.segment_size - 7, seed=4)
    want, ostate, _ = O.Oracle(w, cfg, np.float32).run_diagonal(tokens)
    for dtype in ("bf16", "f32"):
        st = MemoryState.fresh(cfg)
        got, _ = run_diagonal(prepare_weights(w, dtype), cfg, tokens, dtype=dtype, state=st)
        tol = TOL[dtype]
        assert np.isfinite(got).all()
        assert relative_error(got, want) < tol, (dtype, relative_error(got, want))
        assert relative_error(st.A.cpu().numpy(), ostate.A) < tol, dtype
        assert relative_error(st.z.cpu().numpy(), ostate.z) < tol, dtype


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_odd_shapes_match_oracle(dtype):
    """Shapes off every fast path's grid: d 384 (6 heads of 64), d_ff 1000
    (zero-padded to 1024), segment 200 + 24 memory tokens (T 224: partial m- and
    attention tiles), d_mem 32 with DPFP order 2, vocab 777, ragged tail."""
    cfg = ModelConfig(n_layers=3, d_model=384, n_heads=6, d_ff=1000, segment_size=200, num_mem_tokens=24,
                      d_mem=32, dpfp_nu=2, vocab_size=777, eps_assoc=10.0, seed=3)
    w = conditioned_weights(cfg)
    tokens = cli_tokens(cfg, 4 * cfg.segment_size - 37, seed=8)
    want, ostate, _ = O.Oracle(w, cfg, np.float64).run_diagonal(tokens)
    st = MemoryState.fresh(cfg)
    got, _ = run_diagonal(prepare_weights(w, dtype), cfg, tokens, dtype=dtype, state=st)
    assert relative_error(got, want) < TOL[dtype], relative_error(got, want)
    assert relative_error(st.A.cpu().numpy(), ostate.A) < TOL[dtype]
    seq, _ = run_sequential(prepare_weights(w, dtype), cfg, tokens, dtype=dtype)
    assert np.array_equal(seq, got)


@pytest.fixture(scope="module")
def c2_full_depth():
    """The headline model at FULL depth and width: 16 layers, d 2048, 32 heads of
    64, d_ff 8192, segment 1024 + 128 memory tokens, d_mem 64, the bench's
    eps_assoc 100 conditioning; the vocab is cut to 4096 so the f32 CPU oracle
    finishes in about a minute (the LM head does not feed the recurrence).
    3 segments with a ragged tail: 48 cells, 18 wavefront steps, up to 3 members.
    The oracle records every fold's guard inputs (zq, nrm) per token."""
    cfg = ModelConfig(n_layers=16, d_model=2048, n_heads=32, d_ff=8192, segment_size=1024, num_mem_tokens=128,
                      d_mem=64, vocab_size=4096, eps_assoc=100.0, seed=0)
    w = conditioned_weights(cfg)
    tokens = cli_tokens(cfg, 3 * cfg.segment_size - 13, seed=2)
    orc = O.Oracle(w, cfg, np.float32)
    orc.fold_log = []
    want, ostate, _ = orc.run_diagonal(tokens)
    return cfg, w, tokens, want, ostate, orc.fold_log


# A fold token whose |zq| sits within GUARD_BAND of eps_assoc takes the hard branch
# "vbar = |zq| <= eps ? 0 : A phi / zq" (armt/memory.py:107-115) one way or the other
# depending on perturbations of the size bf16 activations introduce (zq = z.phi has
# ~1e-2 relative error after a few layers). When nrm/|zq| is large the two branches
# differ by ~ beta (nrm/|zq|) |A phi| -- a discrete jump in that layer's A that no
# precision short of bit-identical f32 arithmetic avoids. The lockstep audit
# (scripts/lockstep_audit.py, profiles/r2_parity.md) shows the one such cell of this
# fixture (segment 1, layer 9: |zq| within 10% of eps, nrm/|zq| ~ 7): inputs agree to
# 5e-3, A jumps to 0.17 there while z (continuous in zq) stays at 1e-2.
GUARD_BAND, GUARD_GAIN = 0.2, 4.0


def _guard_critical(rows, eps):
    return any(abs(abs(zq) - eps) <= GUARD_BAND * eps and nrm >= GUARD_GAIN * abs(zq) for zq, nrm in rows)


def guard_sensitive_layers(fold_log, eps):
    return {layer for layer, rows in fold_log if _guard_critical(rows, eps)}


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_full_depth_c2_matches_oracle(c2_full_depth, dtype):
    """North-star tolerances at the headline config's depth: f32 mode 1e-4 on
    logits, A and z; bf16 2e-2 on logits (whole run and every segment), z and
    the A of every layer whose folds stay clear of a high-gain guard boundary
    (the oracle decides which, see GUARD_BAND); such layers (4 of 16 here)
    must still be finite and within 0.25."""
    cfg, w, tokens, want, ostate, fold_log = c2_full_depth
    st = MemoryState.fresh(cfg)
    got, trace = run_diagonal(prepare_weights(w, dtype), cfg, tokens, dtype=dtype, state=st)
    tol = TOL[dtype]
    assert np.isfinite(got).all()
    seg = cfg.segment_size
    per_seg = [relative_error(got[s * seg:(s + 1) * seg], want[s * seg:(s + 1) * seg]) for s in range(3)]
    assert max(per_seg) < tol, (dtype, per_seg)
    assert relative_error(got, want) < tol
    A = st.A.cpu().numpy()
    assert relative_error(st.z.cpu().numpy(), ostate.z) < tol, dtype
    per_layer = [relative_error(A[l], ostate.A[l]) for l in range(16)]
    sensitive = guard_sensitive_layers(fold_log, 100.0) if dtype == "bf16" else set()
    assert len(sensitive) <= 4, sensitive   # {5, 6, 9, 10} on this fixture
    for l, e in enumerate(per_layer):
        assert e < (0.25 if l in sensitive else tol), (dtype, l, e, sorted(sensitive))
    keep = [l for l in range(16) if l not in sensitive]
    assert relative_error(A[keep], ostate.A[keep]) < tol
    assert st.updates.tolist() == [3] * 16
    assert trace.steps_executed == 3 + 16 - 1


def test_full_depth_c2_memory_is_live(c2_full_depth):
    """The parity above is only meaningful if the memory changes the outputs:
    with W_k = 0 (nothing stored, every read guarded) the logits of segments
    1-2 must move by well over the f32 tolerance (segment 0 reads an empty
    memory either way, so it must not move at all)."""
    cfg, w, tokens, _, _, _ = c2_full_depth
    live, _ = run_diagonal(prepare_weights(w, "f32"), cfg, tokens, dtype="f32")
    inert_w = replace(w, w_k_mem=np.zeros_like(w.w_k_mem))
    inert, _ = run_diagonal(prepare_weights(inert_w, "f32"), cfg, tokens, dtype="f32")
    seg = cfg.segment_size
    assert np.array_equal(live[:seg], inert[:seg])
    moved = relative_error(live[seg:], inert[seg:])
    assert moved > 1e-2, moved


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_reference_written_container_drives_the_device(dtype):
    """a weight file written by the reference's own
    save_weights (tests/golden/ref_c1_cond_f32.armt) loads here and drives the
    device path to the reference's C1 logits and memory state."""
    import os
    from conftest import GOLDEN
    w = P.load_weights(os.path.join(GOLDEN, "ref_c1_cond_f32.armt"))
    cfg = w.config
    g = golden("c1_cond")
    state = MemoryState.fresh(cfg)
    logits, _ = run_diagonal(w, cfg, g["tokens"], dtype=dtype, state=state)
    assert relative_error(logits, g["logits_f64"]) < TOL[dtype]
    assert relative_error(state.A.cpu().numpy(), g["A_f64"]) < TOL[dtype]


def test_dropin_calls_reuse_prepared_weights_and_replay_one_graph(monkeypatch):
    """run_diagonal(GroupedWeights, ...) as a reference user calls it: weights
    are prepared once per weight object, the first call of a length runs
    eagerly and later calls replay one captured graph of the whole schedule —
    bitwise the eager result, with the caller's memory state carried across
    calls like the eager path; an in-place weight edit is picked up."""
    from paper_2506_05229_b200 import executors as X
    X.clear_caches()
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    w = conditioned_weights(cfg)
    tokens = cli_tokens(cfg, 5 * cfg.segment_size - 7)
    calls = []
    real = X.prepare_weights
    monkeypatch.setattr(X, "prepare_weights", lambda *a, **k: calls.append(1) or real(*a, **k))
    st_e, st_g = MemoryState.fresh(cfg), MemoryState.fresh(cfg)
    eager = [run_diagonal(w, cfg, tokens, state=st_e, graph=False)[0] for _ in range(3)]
    assert len(calls) == 1
    X.clear_caches()
    got = [run_diagonal(w, cfg, tokens, state=st_g)[0] for _ in range(3)]
    assert len(calls) == 2
    run = next(iter(X._RUN_CACHE.values()))
    assert run.runner.graph is not None and run.calls == 3
    for a, b in zip(eager, got):
        assert np.array_equal(a, b)
    assert torch.equal(st_e.A, st_g.A) and torch.equal(st_e.z, st_g.z)
    assert np.array_equal(st_e.updates, st_g.updates)
    w.wo[0] *= 0.5
    changed, _ = run_diagonal(w, cfg, tokens)
    assert len(calls) == 3
    assert not np.array_equal(changed, eager[0])   # fresh state both times: only the weights differ
    X.clear_caches()
