"""Device verify / bench / trace reports (``-m gpu``): the reference's report
documents filled by device runs (armt/cli.py:85-234 counterpart)."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from conftest import C1  # noqa: E402
from fixtures import conditioned_weights  # noqa: E402
from paper_2506_05229_b200.config import ModelConfig  # noqa: E402
from paper_2506_05229_b200.engine import prepare_weights  # noqa: E402
from paper_2506_05229_b200.executors import run_diagonal  # noqa: E402
from paper_2506_05229_b200.reports import bench, trace_document, verify, seeded_tokens  # noqa: E402


def test_device_verify_report_passes_bitwise():
    cfg = ModelConfig(**C1, eps_assoc=1.0)
    rep = verify(conditioned_weights(cfg), [1, 3, 8], precision="both")
    doc = rep.to_json_dict()
    assert doc["passed"]
    assert all(r["rel_error_f32"] == 0.0 and r["rel_error_bf16"] == 0.0 for r in doc["rows"])


def test_device_bench_report_modes():
    cfg = ModelConfig(**C1, eps_assoc=1.0)
    prep = prepare_weights(conditioned_weights(cfg), "bf16")
    rep = bench(prep, [4 * cfg.segment_size], copies=2, repeat=2)
    doc = rep.to_json_dict()
    assert [r["mode"] for r in doc["rows"]] == ["sequential", "diagonal", "minibatch"]
    assert doc["rows"][0]["speedup_vs_sequential"] == 1.0
    assert all(r["wall_seconds"] > 0 for r in doc["rows"])


def test_device_trace_document():
    cfg = ModelConfig(**C1, eps_assoc=1.0)
    prep = prepare_weights(conditioned_weights(cfg), "bf16")
    _, tr = run_diagonal(prep, cfg, seeded_tokens(cfg, 3 * cfg.segment_size), timed=True)
    doc = trace_document(tr)
    assert len(doc["steps"]) == 3 + cfg.n_layers - 1
    assert all(s["duration_ns"] > 0 for s in doc["steps"])
