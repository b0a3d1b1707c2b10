"""The driver's bench.py contract: one JSON line with the keys the round-end
harness reads, for the reference arm (CPU, the reference's own numba cores from
baseline/_ref) and for the device arm (``-m gpu``, a 4-segment C2 run)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRIC = "tokens/sec for one 131k-token seq, LLaMA-1B ARMT seg1024, 1/2/4/8 B200"


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:]
    return json.loads(lines[-1])


def _check_common(d):
    assert d["metric"] == METRIC
    assert d["unit"] == "tokens/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["n_gpus"] == 1 and d["steps"] >= 1
    assert d["config"]["workload"].startswith("C2:")
    e2e = d["e2e"]
    assert e2e["unit"] == "tokens/s" and e2e["value"] > 0
    assert e2e["h2d_bytes_per_step"] >= 0 and e2e["d2h_bytes_per_step"] >= 0


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "armt")),
                    reason="reference arm not installed (build() installs it into baseline/_ref)")
def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], timeout=900)
    _check_common(d)
    assert d["impl"] == "reference"
    cpu = d["cpu_baseline"]
    assert cpu["kind"] == "reference" and cpu["cores"] >= 1 and cpu["sample"]
    assert cpu["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_device_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    d = _run(["--steps", "1", "--warmup", "3", "--segments", "4", "--no-cpu-baseline"], timeout=1200)
    _check_common(d)
    assert d["dtype"] == "bf16" and d["scaling"] in ("weak", "strong") and d["data"].startswith("synthetic")
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s" and rf["peak"] > 0
    assert 0 < rf["frac"] == pytest.approx(rf["achieved"] / rf["peak"])
    assert d["gpu_launches"] > 0
    assert d["clocks"]["samples"] >= 0 and "reasons" in d["clocks"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["sequential_value"] > 0 and d["diag_over_seq"] == pytest.approx(d["value"] / d["sequential_value"])
    assert d["e2e_reference_api"]["value"] > 0
