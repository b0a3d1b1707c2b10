"""Scheduler bookkeeping pinned to the reference (CPU, bit-exact).

Ports of the reference's pkg/tests/test_scheduler.py (construction,
validation violation lists, optimality oracle) against this package's
``scheduler`` module, plus the device executors' step plans
(``diagonal_plan`` / ``sequential_plan``) checked node for node against
traces recorded by running the reference's own run_diagonal / run_sequential
(tests/golden/traces.npz, scripts/make_golden.py), including its
``shuffle_seed`` member-order audit hook (armt/executors.py:192-195).
"""

import numpy as np
import pytest

from conftest import golden
from paper_2506_05229_b200.errors import InputError
from paper_2506_05229_b200.scheduler import (MAX_ORACLE_NODES, DiagonalSchedule, Node, build_diagonal_schedule,
                                             diagonal_members, min_groups_oracle, validate_schedule)

torch = pytest.importorskip("torch")   # executors import torch (plans themselves are host-only)
from paper_2506_05229_b200.executors import diagonal_plan, sequential_plan  # noqa: E402


# ---------------------------------------------------------------- Node (test_scheduler.py:14-19)
def test_node_predecessors():
    assert Node(0, 0).predecessors() == []
    assert Node(0, 2).predecessors() == [Node(0, 1)]
    assert Node(3, 0).predecessors() == [Node(2, 0)]
    assert set(Node(2, 2).predecessors()) == {Node(1, 2), Node(2, 1)}


# ---------------------------------------------------------------- construction (:26-64)
def test_diagonal_groups_for_4x3_by_hand():
    sched = build_diagonal_schedule(4, 3)
    expected = [{(0, 0)}, {(0, 1), (1, 0)}, {(0, 2), (1, 1), (2, 0)}, {(1, 2), (2, 1), (3, 0)},
                {(2, 2), (3, 1)}, {(3, 2)}]
    assert [{(n.segment, n.layer) for n in g} for g in sched.groups] == expected
    assert len(sched) == 6
    assert sched.max_group_size() == 3


@pytest.mark.parametrize("S,L", [(1, 1), (1, 5), (5, 1), (2, 2)])
def test_diagonal_degenerate_grids(S, L):
    sched = build_diagonal_schedule(S, L)
    assert len(sched) == S + L - 1
    assert sum(len(g) for g in sched.groups) == S * L
    if S == 1 or L == 1:
        assert sched.max_group_size() == 1


def test_every_node_in_its_earliest_group():
    sched = build_diagonal_schedule(6, 4)
    for i, group in enumerate(sched.groups):
        assert all(n.segment + n.layer == i for n in group)


def test_json_obj_sorted_and_plain():
    assert build_diagonal_schedule(3, 2).to_json_obj() == [[[0, 0]], [[0, 1], [1, 0]], [[1, 1], [2, 0]], [[2, 1]]]


@pytest.mark.parametrize("S,L", [(0, 3), (3, 0), (-1, 1)])
def test_build_rejects_empty_grids(S, L):
    with pytest.raises(InputError):
        build_diagonal_schedule(S, L)


def test_c2_group_sizes():
    """The headline grid (S=128, L=16): 143 groups ramping 1..16, 113 full groups, Σ = 2048."""
    sched = build_diagonal_schedule(128, 16)
    sizes = [len(g) for g in sched.groups]
    assert len(sizes) == 143 and sum(sizes) == 2048
    assert sizes[:16] == list(range(1, 17)) and sizes[-16:] == list(range(16, 0, -1))
    assert sizes.count(16) == 113


# ---------------------------------------------------------------- validation (:70-126)
@pytest.mark.parametrize("S,L", [(1, 1), (4, 3), (7, 2), (5, 5)])
def test_built_schedules_validate(S, L):
    check = validate_schedule(build_diagonal_schedule(S, L), S, L)
    assert check.ok and check.violations == []


def test_sequential_row_major_validates():
    groups = [[(s, l)] for s in range(4) for l in range(3)]
    assert validate_schedule(groups, 4, 3).ok


def test_same_group_dependency_flagged():
    check = validate_schedule([[(0, 0), (0, 1)], [(1, 0)], [(1, 1)]], 2, 2)
    assert not check.ok
    assert any("(0,0) -> (0,1)" in v for v in check.violations)


def test_reversed_layers_flagged():
    check = validate_schedule([[(0, 1)], [(0, 0)]], 1, 2)
    assert not check.ok
    assert any("broken" in v for v in check.violations)


def test_duplicate_node_flagged():
    check = validate_schedule([[(0, 0)], [(0, 0)], [(0, 1)]], 1, 2)
    assert not check.ok
    assert any("appears in groups 0 and 1" in v for v in check.violations)


def test_missing_node_flagged():
    check = validate_schedule([[(0, 0)]], 1, 2)
    assert not check.ok
    assert any("never scheduled" in v for v in check.violations)


def test_out_of_bounds_node_flagged():
    check = validate_schedule([[(0, 0)], [(0, 1)], [(5, 0)]], 1, 2)
    assert not check.ok
    assert any("out of grid bounds" in v for v in check.violations)


def test_violation_messages_are_exact_and_sorted():
    """Same message text and order as armt/scheduler.py:94-130 (sorted list)."""
    check = validate_schedule([[(0, 1), (0, 0)], [(0, 0)], [(3, 3)]], 1, 3)
    assert check.violations == sorted([
        "edge (0,0) -> (0,1) broken: predecessor in group 0, node in group 0",
        "node (0,0) appears in groups 0 and 1",
        "node (0,2) never scheduled",
        "node (3,3) out of grid bounds",
    ])


def test_validate_accepts_node_objects():
    sched = DiagonalSchedule(2, 2, [{Node(0, 0)}, {Node(0, 1), Node(1, 0)}, {Node(1, 1)}])
    assert validate_schedule(sched, 2, 2).ok


# ---------------------------------------------------------------- optimality oracle (:132-152)
@pytest.mark.parametrize("S,L,expected", [(1, 1, 1), (1, 7, 7), (7, 1, 7), (4, 3, 6), (16, 16, 31),
                                          (128, 16, 143)])
def test_oracle_frozen_values(S, L, expected):
    assert min_groups_oracle(S, L) == expected


def test_oracle_matches_diagonal_length_on_small_grids():
    for S in range(1, 9):
        for L in range(1, 9):
            assert min_groups_oracle(S, L) == len(build_diagonal_schedule(S, L)) == S + L - 1


def test_oracle_scale_bound():
    big = int(MAX_ORACLE_NODES ** 0.5) + 1
    with pytest.raises(InputError):
        min_groups_oracle(big, big)


@pytest.mark.parametrize("S,L", [(0, 3), (3, 0)])
def test_oracle_rejects_empty_grids(S, L):
    with pytest.raises(InputError):
        min_groups_oracle(S, L)


# ---------------------------------------------------------------- device plans vs reference traces
def _flat(plan):
    return np.array([[n.segment, n.layer] for st in plan.steps for n in st.nodes], np.int64).reshape(-1, 2)


def _counts(plan):
    return np.array([len(st.nodes) for st in plan.steps], np.int64)


@pytest.mark.parametrize("S,L", [(4, 3), (3, 2), (1, 5), (5, 1), (7, 4)])
def test_diagonal_plan_equals_reference_trace(S, L):
    g = golden("traces")
    plan = diagonal_plan(S, L)
    assert np.array_equal(_flat(plan), g[f"nodes_{S}x{L}"])
    assert np.array_equal(_counts(plan), g[f"counts_{S}x{L}"])
    # the plan's groups are the schedule's groups; members in ascending layer order
    sched = build_diagonal_schedule(S, L)
    for i, st in enumerate(plan.steps):
        assert set(st.nodes) == sched.groups[i]
        assert st.nodes == diagonal_members(i, S, L)
    assert validate_schedule([st.nodes for st in plan.steps], S, L).ok


@pytest.mark.parametrize("S,L,seed", [(4, 3, 7), (7, 4, 123), (9, 6, 2024), (16, 16, 5)])
def test_shuffled_diagonal_plan_replays_reference_rng(S, L, seed):
    """shuffle_seed permutes the in-flight members with the reference's exact
    RNG call sequence; the recorded member order must match node for node."""
    g = golden("traces")
    plan = diagonal_plan(S, L, shuffle_seed=seed)
    assert np.array_equal(_flat(plan), g[f"shuf_nodes_{S}x{L}_seed{seed}"])
    assert np.array_equal(_counts(plan), g[f"shuf_counts_{S}x{L}_seed{seed}"])
    assert validate_schedule([st.nodes for st in plan.steps], S, L).ok
    # slots follow the segment, so a permutation only reorders the members
    for st in plan.steps:
        assert st.slots == [n.segment % plan.n_slots for n in st.nodes]
        assert st.layers == [n.layer for n in st.nodes]


def test_sequential_plan_equals_reference_trace():
    g = golden("traces")
    plan = sequential_plan(3, 4)
    assert np.array_equal(_flat(plan), g["seq_nodes_3x4"])
    assert all(len(st.nodes) == 1 for st in plan.steps)


def test_plan_slots_never_alias_in_flight_segments():
    """Two members of a step never share an activation slot, and a slot is not
    re-embedded while its previous segment is still in flight."""
    for S, L in [(5, 3), (20, 16), (128, 16), (3, 8)]:
        plan = diagonal_plan(S, L)
        live = {}
        for st in plan.steps:
            if st.enter is not None:
                seg, slot = st.enter
                assert slot not in live, (S, L, seg, slot)
                live[slot] = seg
            assert len(set(st.slots)) == len(st.slots)
            for n, slot in zip(st.nodes, st.slots):
                assert live[slot] == n.segment
            for seg, slot in st.exits:
                assert live.pop(slot) == seg
        assert not live
