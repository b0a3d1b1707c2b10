"""Fixture builders shared by CPU and GPU tests (same recipe as
scripts/make_golden.py, re-implemented on this package's initializer)."""

from dataclasses import replace

import numpy as np

from paper_2506_05229_b200.config import ModelConfig
from paper_2506_05229_b200.weights import init_weights, round_to_bf16


def conditioned_weights(cfg: ModelConfig, damp: float = 1.0 / 32):
    """SURVEY Appendix B conditioning + bf16-grid weights."""
    w = init_weights(cfg)
    w = replace(w, w_v_mem=w.w_v_mem * damp)
    return w.map_arrays(round_to_bf16)


def cli_tokens(cfg: ModelConfig, n: int, seed: int = 0):
    """armt/cli.py:45-49."""
    return np.random.default_rng([seed, n]).integers(0, cfg.vocab_size, n, dtype=np.int64)
