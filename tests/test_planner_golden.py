"""Product planner vs golden vectors produced by the REFERENCE planner
(tests/golden/planner_golden.json, generator committed beside it). Runs on
any box — this is the schedule/partition parity gate on the GPU box, where
/root/reference does not exist.
"""
import hashlib
import json
import os

import pytest

from paper_2604_27085_b200.planner import COST_DTYPE, Planner

import numpy as np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "planner_golden.json")
with open(GOLDEN) as f:
    DATA = json.load(f)


def _digest(arr):
    return hashlib.sha256(arr.tobytes()).hexdigest()[:32]


@pytest.mark.parametrize("case", DATA["cases"],
                         ids=[f"{c['model']}-s{c['seq']}-N{c['N']}" for c in DATA["cases"]])
def test_case(product: Planner, case):
    costs = np.array([tuple(c) for c in case["costs"]], dtype=COST_DTYPE)
    # the cost table itself, recomputed from the repo's configs
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    m = product.load_model(os.path.join(root, "configs", "models", case["model"] + ".json"))
    g = product.load_gpu(os.path.join(root, "configs", "gpus", "b200.json"))
    assert np.array_equal(product.layer_costs(m, case["seq"], 1, g, True), costs)

    plan = product.optimal_partition(costs, case["N"], case["M"])
    assert [[r.first, r.last] for r in plan.fwd_stages] == case["plan"]["fwd"]
    assert [plan.fused_stage.first, plan.fused_stage.last] == case["plan"]["fused"]
    assert [[r.first, r.last] for r in plan.bwd_stages] == case["plan"]["bwd"]
    assert plan.t_max_ns == case["plan"]["t_max_ns"]
    assert plan.objective == case["plan"]["objective"]
    durs = product.slot_durations(plan, costs)
    assert durs == case["slot_durs"]
    for kind, barrier in (("roundpipe-sync", True), ("roundpipe", False)):
        exp = case[kind]
        s = product.synthesize(kind, case["N"], case["M"], case["M_R"],
                               case["iters"] if kind == "roundpipe" else 1, durs)
        assert len(s.tasks) == exp["n_tasks"]
        assert s.tasks[:8].tolist() == [tuple(t) for t in exp["first_tasks"]]
        assert _digest(s.tasks) == exp["tasks_sha"]
        rep = product.simulate(s, barrier)
        assert _digest(rep.timeline) == exp["timeline_sha"]
        assert (rep.makespan_ns, rep.bubble_num, rep.bubble_den) == \
            (exp["makespan_ns"], exp["bubble_num"], exp["bubble_den"])
        if "interior" in exp:
            lo, hi = exp["interior_window"]
            assert list(product.interior_bubble(rep.timeline, case["N"], lo, hi)) == \
                exp["interior"]
    assert [list(v) for v in product.stage_feasibility(plan, costs, g, case["M"])] == \
        case["feasibility"]
    pr = case["protocol"]
    proto = product.build_protocol(pr["L"], pr["T"])
    assert len(proto.actions) == pr["n_actions"] and len(proto.edges) == pr["n_edges"]
    edges = [list(e) for e in proto.edges]
    assert hashlib.sha256(json.dumps(edges).encode()).hexdigest()[:32] == pr["edges_sha"]


def test_protocol_makespans(product: Planner):
    for key, val in DATA["protocol_makespans"].items():
        L, T, mode = key.split(",")
        assert product.protocol_makespan(int(L), int(T), mode) == val, key


def test_reference_known_answers(product: Planner):
    """Known-answer tests from the reference's own suites."""
    from tests.test_planner_parity import rand_costs  # noqa: F401
    c = np.zeros(2, dtype=COST_DTYPE)
    c["t_fwd_ns"], c["t_bwd_ns"], c["param_bytes"] = [1, 2], [3, 6], 1
    assert product.candidate_tmax(c) == [1, 2, 3, 6, 9]  # partitioner_tests.cpp:82-87
    one = np.zeros(1, dtype=COST_DTYPE)
    one[0] = (7, 21, 1, 0, 0)
    p = product.optimal_partition(one, 1, 1)  # partitioner_tests.cpp:101-110
    assert p.num_slots() == 1 and p.t_max_ns == 21
    s = product.synthesize("roundpipe-sync", 4, 16, 8, 1, [1000] * 6)
    rep = product.simulate(s)  # simulator_tests.cpp:60-69 → 12/108
    assert rep.bubble_num * 108 == 12 * rep.bubble_den
    tp = product.plan([(f"t{i}", s_) for i, s_ in enumerate([9, 7, 6, 5, 4])], 3, 100)
    assert sorted(tp.window_totals) == [9, 11, 11]  # transfer_planner_tests.cpp:28-37
    assert product.optimal_makespan([9, 7, 6, 5, 4], 3) == 11
    for drop in range(1, 5):  # consistency_tests.cpp:20-40
        v = product.check_all_interleavings(2, 2, "event-per-layer", drop)
        assert not v.ok and v.violated_constraint == drop
        assert v.witness[-1][0] == {1: 3, 2: 0, 3: 4, 4: 1}[drop]
