"""Machine-readable verify / bench / trace reports for the device path.

Counterpart of the reference's report layer (armt/reports.py:1-138) and of
the CLI commands that fill it (armt/cli.py:85-234, ``cmd_verify`` /
``cmd_bench`` / ``cmd_trace``): the same document shapes (field names, CSV
headers, tolerance gates) so tooling that reads the reference's reports reads
these. Differences are device facts, stated in the schemas shipped in
``schemas/``: precisions are the device ones (``f32`` parity mode and
``bf16``; f64 stays in the oracle, so ``rel_error_f64`` is null), the bench
rows add ``tokens_per_second``, and traces may be ``minibatch`` (one node
per copy-step). Every document is validated against its schema before it is
returned, as in the reference (armt/reports.py:36-45).
"""

from __future__ import annotations

import io
import json
import math
import os
import statistics
import time
from dataclasses import dataclass, field
from datetime import datetime, timezone

import numpy as np

from .config import ModelConfig
from .errors import InputError

# diagonal-vs-sequential gates (armt/reports.py:21-23). On the device both
# schedules run the same member-lane-independent kernels, so the measured
# error is 0.0 (bitwise); the gates are kept for drop-in semantics.
TOLERANCES = {"f32": 1e-3, "f64": 1e-12, "bf16": 2e-2}

VERIFY_CSV_HEADER = "segments,rel_error_f32,rel_error_f64"
BENCH_CSV_HEADER = ("mode,threads,seq_len,segments,wall_seconds,"
                    "seconds_per_segment,speedup_vs_sequential")

_SCHEMA_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "schemas")


def _utc_now() -> str:
    return datetime.now(timezone.utc).isoformat()


def load_schema(name: str) -> dict:
    with open(os.path.join(_SCHEMA_DIR, f"{name}.schema.json")) as fh:
        return json.load(fh)


def validate_report(obj: dict, schema_name: str) -> None:
    """Schema check before a document leaves the process (armt/reports.py:36-45)."""
    import jsonschema
    try:
        jsonschema.validate(obj, load_schema(schema_name))
    except jsonschema.ValidationError as exc:
        raise InputError(f"{schema_name} report fails its schema: {exc.message}") from exc


def config_echo(config: ModelConfig) -> dict:
    from dataclasses import asdict
    return {k: v for k, v in asdict(config).items()}


def _device_name() -> str:
    import torch
    return torch.cuda.get_device_name() if torch.cuda.is_available() else "none"


# =========================================================================
# Verify
# =========================================================================

@dataclass
class VerifyRow:
    segments: int
    rel_error_f32: float | None
    rel_error_f64: float | None = None
    rel_error_bf16: float | None = None


@dataclass
class VerifyReport:
    config: dict
    precision: str                    # f32 | bf16 | both
    rows: list[VerifyRow]
    passed: bool
    tolerance_f32: float = TOLERANCES["f32"]
    tolerance_f64: float = TOLERANCES["f64"]
    tolerance_bf16: float = TOLERANCES["bf16"]
    device: str = ""
    timestamp: str = field(default_factory=_utc_now)

    def to_json_dict(self) -> dict:
        doc = {
            "config": self.config, "precision": self.precision,
            "tolerance_f32": self.tolerance_f32, "tolerance_f64": self.tolerance_f64,
            "tolerance_bf16": self.tolerance_bf16, "device": self.device,
            "rows": [{"segments": r.segments, "rel_error_f32": r.rel_error_f32,
                      "rel_error_f64": r.rel_error_f64, "rel_error_bf16": r.rel_error_bf16} for r in self.rows],
            "passed": self.passed, "timestamp": self.timestamp,
        }
        validate_report(doc, "verify")
        return doc

    def to_csv(self) -> str:
        out = io.StringIO()
        out.write(VERIFY_CSV_HEADER + "\n")
        for r in self.rows:
            f32 = "" if r.rel_error_f32 is None else repr(r.rel_error_f32)
            f64 = "" if r.rel_error_f64 is None else repr(r.rel_error_f64)
            out.write(f"{r.segments},{f32},{f64}\n")
        return out.getvalue()


def seeded_tokens(config: ModelConfig, n: int, seed: int = 0) -> np.ndarray:
    """The reference's synthetic token convention (armt/cli.py:45-49)."""
    return np.random.default_rng([seed, n]).integers(0, config.vocab_size, n, dtype=np.int64)


def verify(weights, segments: list[int], precision: str = "both", device=None) -> VerifyReport:
    """cmd_verify (armt/cli.py:85-122) on the device: diagonal vs sequential
    relative Frobenius error of the logits per segment count and precision."""
    from .executors import relative_error, run_diagonal, run_sequential
    config = weights.config
    if precision not in ("f32", "bf16", "both"):
        raise InputError(f"precision must be f32, bf16 or both, got {precision!r}")
    precisions = ["f32", "bf16"] if precision == "both" else [precision]
    rows, failures = [], []
    for S in sorted(set(segments)):
        if S < 1:
            raise InputError(f"segment counts must be >= 1, got {S}")
        tokens = seeded_tokens(config, S * config.segment_size)
        errs: dict[str, float | None] = {"f32": None, "bf16": None}
        for prec in precisions:
            base, _ = run_sequential(weights, config, tokens, dtype=prec, device=device)
            diag, _ = run_diagonal(weights, config, tokens, dtype=prec, device=device)
            err = relative_error(diag, base)
            errs[prec] = err
            if not err <= TOLERANCES[prec]:
                failures.append(f"segments={S} {prec}: rel_error {err:.3e} exceeds {TOLERANCES[prec]:.1e}")
        rows.append(VerifyRow(segments=S, rel_error_f32=errs["f32"], rel_error_f64=None,
                              rel_error_bf16=errs["bf16"]))
    return VerifyReport(config=config_echo(config), precision=precision, rows=rows, passed=not failures,
                        device=_device_name())


# =========================================================================
# Bench
# =========================================================================

@dataclass
class BenchRow:
    mode: str                         # sequential | diagonal | minibatch
    threads: int                      # minibatch: copies; otherwise 1 (one device stream)
    seq_len: int
    segments: int
    wall_seconds: float
    seconds_per_segment: float
    speedup_vs_sequential: float
    tokens_per_second: float | None = None


@dataclass
class BenchReport:
    config: dict
    environment: dict
    rows: list[BenchRow]

    def to_json_dict(self) -> dict:
        doc = {
            "config": self.config, "environment": self.environment,
            "rows": [{k: v for k, v in (("mode", r.mode), ("threads", r.threads), ("seq_len", r.seq_len),
                                        ("segments", r.segments), ("wall_seconds", r.wall_seconds),
                                        ("seconds_per_segment", r.seconds_per_segment),
                                        ("speedup_vs_sequential", r.speedup_vs_sequential),
                                        ("tokens_per_second", r.tokens_per_second)) if v is not None}
                     for r in self.rows],
        }
        validate_report(doc, "bench")
        return doc

    def to_csv(self) -> str:
        out = io.StringIO()
        out.write(BENCH_CSV_HEADER + "\n")
        for r in self.rows:
            out.write(f"{r.mode},{r.threads},{r.seq_len},{r.segments},{r.wall_seconds!r},"
                      f"{r.seconds_per_segment!r},{r.speedup_vs_sequential!r}\n")
        return out.getvalue()


def _median_wall(fn, repeat: int) -> float:
    """One discarded warm-up, then the median of ``repeat`` device-synchronised
    runs (armt/cli.py:129-136), timed with CUDA events."""
    import torch
    fn()
    torch.cuda.synchronize()
    walls = []
    for _ in range(repeat):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        walls.append(a.elapsed_time(b) / 1e3)
    return statistics.median(walls)


def bench(prepared, seq_lens: list[int], modes=("sequential", "diagonal", "minibatch"), copies: int = 4,
          repeat: int = 3) -> BenchReport:
    """cmd_bench (armt/cli.py:155-234) on the device. Each sequence length is
    compiled once per schedule into a CUDA-graph ``Session`` and replayed;
    minibatch runs ``copies`` lockstep copies of the stream (seconds per
    segment divide by segments x copies, as in the reference)."""
    import torch
    from .engine import MemoryState
    from .executors import Runner, Session, minibatch_plan
    config = prepared.config
    if repeat < 1:
        raise InputError(f"repeat must be >= 1, got {repeat}")
    rows = []
    for n in seq_lens:
        if n < 1:
            raise InputError(f"seq_len values must be >= 1, got {n}")
        S = math.ceil(n / config.segment_size)
        tokens = torch.as_tensor(seeded_tokens(config, n)).to(prepared.device)
        walls = {}
        for mode in ("sequential",) + tuple(m for m in modes if m != "sequential"):
            if mode in ("sequential", "diagonal"):
                sess = Session(prepared, n, schedule=mode)
                sess._load_ids(tokens)
                sess.warm()
                walls[mode] = _median_wall(sess.forward, repeat)
                del sess
            elif mode == "minibatch":
                runner = Runner(prepared, minibatch_plan(S, config.n_layers, copies))
                runner.ids[:n].copy_(tokens)
                st = MemoryState.fresh(config, prepared.device, n_layers=copies * config.n_layers)
                runner.run(st)
                runner.capture(st, reset_state=True)
                walls[mode] = _median_wall(runner.replay, repeat)
                del runner
            else:
                raise InputError(f"unknown bench mode {mode!r}")
            torch.cuda.empty_cache()
        for mode in modes:
            k = copies if mode == "minibatch" else 1
            w = walls[mode]
            rows.append(BenchRow(mode=mode, threads=k, seq_len=n, segments=S, wall_seconds=w,
                                 seconds_per_segment=w / (S * k),
                                 speedup_vs_sequential=walls["sequential"] / w,
                                 tokens_per_second=n * k / w))
    env = {"precision": prepared.dtype_name, "host_workers": 1, "device": _device_name(), "timestamp": _utc_now()}
    return BenchReport(config=config_echo(config), environment=env, rows=rows)


# =========================================================================
# Trace
# =========================================================================

def trace_document(trace) -> dict:
    """cmd_trace (armt/cli.py): the ExecutionTrace JSON, schema-checked."""
    doc = trace.to_json_dict()
    validate_report(doc, "trace")
    return doc
