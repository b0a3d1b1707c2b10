"""Report documents (armt/reports.py counterpart) and the minibatch plan: host
logic, CPU-only. The device runs that fill them are in test_gpu_reports.py."""

import pytest

from conftest import C1
from paper_2506_05229_b200.config import ModelConfig
from paper_2506_05229_b200.errors import InputError
from paper_2506_05229_b200.executors import ExecutionTrace, TraceEvent, minibatch_plan, sequential_plan
from paper_2506_05229_b200.reports import (BENCH_CSV_HEADER, VERIFY_CSV_HEADER, BenchReport, BenchRow,
                                           VerifyReport, VerifyRow, config_echo, trace_document,
                                           validate_report)
from paper_2506_05229_b200.scheduler import Node


def test_verify_report_shape_and_csv():
    cfg = ModelConfig(**C1)
    rep = VerifyReport(config=config_echo(cfg), precision="both",
                       rows=[VerifyRow(2, 0.0, None, 0.0), VerifyRow(8, 0.0, None, 0.0)], passed=True, device="x")
    doc = rep.to_json_dict()
    assert doc["rows"][1]["segments"] == 8 and doc["rows"][0]["rel_error_f64"] is None
    assert rep.to_csv().splitlines()[0] == VERIFY_CSV_HEADER
    assert rep.to_csv().splitlines()[1] == "2,0.0,"
    with pytest.raises(InputError):
        VerifyReport(config={}, precision="f64x", rows=[VerifyRow(1, 0.0)], passed=True).to_json_dict()


def test_bench_report_shape_and_csv():
    rows = [BenchRow("sequential", 1, 512, 8, 2.0, 0.25, 1.0, 256.0),
            BenchRow("minibatch", 4, 512, 8, 3.0, 3.0 / 32, 2.0 / 3.0, 682.0)]
    rep = BenchReport(config={}, environment={"precision": "bf16", "host_workers": 1, "timestamp": "t"}, rows=rows)
    doc = rep.to_json_dict()
    assert [r["mode"] for r in doc["rows"]] == ["sequential", "minibatch"]
    assert rep.to_csv().splitlines()[0] == BENCH_CSV_HEADER
    bad = BenchReport(config={}, environment={"precision": "bf16", "host_workers": 1, "timestamp": "t"},
                      rows=[BenchRow("turbo", 1, 1, 1, 1.0, 1.0, 1.0)])
    with pytest.raises(InputError):
        bad.to_json_dict()


def test_trace_document_validates():
    tr = ExecutionTrace("diagonal", [TraceEvent(0, [Node(0, 0)], [0], 5), TraceEvent(1, [Node(1, 0), Node(0, 1)], [0, 0], 7)], 12)
    doc = trace_document(tr)
    assert doc["steps"][1]["nodes"] == [[1, 0], [0, 1]]
    with pytest.raises(InputError):
        validate_report({"schedule_kind": "diagonal", "steps": [], "total_ns": 0}, "trace")


@pytest.mark.parametrize("S,L,B", [(3, 2, 1), (4, 5, 3), (1, 1, 8)])
def test_minibatch_plan_is_lockstep_sequential(S, L, B):
    plan = minibatch_plan(S, L, B)
    seq = sequential_plan(S, L)
    assert len(plan.steps) == len(seq.steps) == S * L
    for st, sq in zip(plan.steps, seq.steps):
        assert st.nodes == [sq.nodes[0]] * B
        assert st.layers == [sq.layers[0]] * B and st.slots == list(range(B))
        assert st.state_layers == [b * L + sq.layers[0] for b in range(B)]
        if sq.enter is not None:
            assert st.enters == [(sq.enter[0], b) for b in range(B)]
        if sq.exits:
            assert st.exit_rows == [b * S + sq.exits[0][0] for b in range(B)]
    with pytest.raises(InputError):
        minibatch_plan(2, 2, 0)
