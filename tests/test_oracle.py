"""Pin the NumPy oracle to the reference's own outputs (golden vectors made
by scripts/make_golden.py from /root/reference) and to the reference's
known-answer tests. CPU only."""

import hashlib

import numpy as np
import pytest

import armt_oracle as O
from conftest import C1, MID, SMALL, golden
from fixtures import cli_tokens, conditioned_weights
from paper_2506_05229_b200.config import ModelConfig
from paper_2506_05229_b200.weights import init_weights
from dataclasses import replace


def digest(w):
    h = hashlib.sha256()
    for name in w.NAMES:
        h.update(np.ascontiguousarray(getattr(w, name), np.float64).tobytes())
    return h.hexdigest()


def test_init_weights_bitwise_equal_reference():
    # armt/weights.py:98-138 draw order: identical seeds give identical bytes.
    assert digest(init_weights(ModelConfig(**SMALL))) == str(golden("small_ref")["digest"])
    assert digest(init_weights(ModelConfig(**C1, eps_assoc=1.0))) == str(golden("c1_cond")["digest"])


def test_dpfp_known_answers():
    # pkg/tests/test_memory.py:25-33
    assert np.array_equal(O.dpfp(np.array([2.0]), 3), [0, 0, 4, 0, 0, 0])
    assert np.array_equal(O.dpfp(np.array([-2.0]), 3), [0, 0, 0, 4, 0, 0])
    assert np.array_equal(O.dpfp(np.array([1.0, -2.0]), 1), [0, 0, 0, 2])


def test_oracle_matches_reference_small_fixture():
    g = golden("small_ref")
    cfg = ModelConfig(**SMALL)
    raw = init_weights(cfg)
    w = replace(raw, w_v_mem=raw.w_v_mem * 0.03125)
    orc = O.Oracle(w, cfg, np.float64)
    logits, st, _ = orc.run_sequential(g["tokens"])
    assert O.relative_error(logits, g["logits"]) < 1e-12
    assert O.relative_error(st.A, g["A"]) < 1e-12
    assert np.array_equal(st.updates, g["updates"])


@pytest.mark.parametrize("dt,tol", [("f64", 1e-7), ("f32", 2e-5)])
def test_oracle_matches_reference_c1(dt, tol):
    g = golden("c1_cond")
    cfg = ModelConfig(**C1, eps_assoc=1.0)
    w = conditioned_weights(cfg)
    orc = O.Oracle(w, cfg, np.float64 if dt == "f64" else np.float32)
    logits, st, nodes = orc.run_diagonal(g["tokens"])
    assert O.relative_error(logits, g[f"logits_{dt}"]) < tol
    assert O.relative_error(st.A, g[f"A_{dt}"]) < tol
    assert O.relative_error(st.z, g[f"z_{dt}"]) < tol
    flat = np.array([x for step in nodes for x in step])
    assert np.array_equal(flat, g["nodes"])


def test_oracle_matches_reference_mid():
    g = golden("mid_cond")
    cfg = ModelConfig(**MID, eps_assoc=10.0)
    w = conditioned_weights(cfg)
    logits, st, _ = O.Oracle(w, cfg).run_sequential(g["tokens"])
    assert logits.shape == g["logits"].shape
    assert O.relative_error(logits, g["logits"]) < 1e-6
    assert O.relative_error(st.A, g["A"]) < 1e-6


def test_oracle_memory_is_live_on_c1():
    # The conditioned fixture must keep the memory path observable.
    g = golden("c1_cond")
    assert O.relative_error(g["logits_inert_f64"], g["logits_f64"]) > 0.05


def test_oracle_per_core_goldens():
    g = golden("ops_c1")
    cfg = ModelConfig(**C1, eps_assoc=1.0)
    w = conditioned_weights(cfg)
    orc = O.Oracle(w, cfg, np.float64)
    for gi, l in enumerate([0, 1]):
        x = g["x_f64"][gi]
        lw = orc.layers[l]
        xr = O.retrieve(g["A0_f64"][l], g["z0_f64"][l], x, lw.w_q_assoc, cfg.dpfp_nu, orc.eps)
        assert O.relative_error(xr, g["retrieved_f64"][gi]) < 1e-12
        y = O.block(x, lw, cfg.n_heads, cfg.eps_norm, orc.cos, orc.sin)
        assert O.relative_error(y, g["forward_f64"][gi]) < 1e-12
        A, z = g["A0_f64"][l].copy(), g["z0_f64"][l].copy()
        O.fold(A, z, y[cfg.segment_size:], lw, cfg.dpfp_nu, orc.eps)
        assert O.relative_error(A, g["A1_f64"][l]) < 1e-12
        assert O.relative_error(z, g["z1_f64"][l]) < 1e-12


def test_relative_error_values():
    # pkg/tests/test_executors.py:240-246 semantics
    assert O.relative_error(np.zeros(3), np.zeros(3)) == 0.0
    assert O.relative_error(np.ones(3), np.zeros(3)) == float("inf")
    assert O.relative_error(np.array([1.0, 1.0]), np.array([1.0, 0.0])) == 1.0
