"""Shared test plumbing.

``-m "not gpu"`` runs here (no GPU): oracle vs golden vectors, host logic,
C-ABI symbol exports. ``-m gpu`` runs on a B200: device parity against the
oracle and the reference's golden vectors.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


C1 = dict(n_layers=2, d_model=128, n_heads=4, d_ff=512, segment_size=64,
          num_mem_tokens=16, d_mem=16, vocab_size=256)
MID = dict(n_layers=4, d_model=256, n_heads=4, d_ff=512, segment_size=128,
           num_mem_tokens=16, d_mem=16, vocab_size=512)
SMALL = dict(n_layers=3, d_model=16, n_heads=2, d_ff=32, segment_size=6,
             num_mem_tokens=2, d_mem=4, vocab_size=50, seed=7)
