"""Generate tests/golden/planner_golden.json from the REFERENCE planner.

Run in the build container (needs oracle/_ref/libref_planner.so, i.e.
/root/reference at build time):  python tests/golden/make_planner_golden.py
The fixture pins, for the B200 configs this repo runs (tiny / Qwen3-1.7B /
Qwen3-8B / Qwen3-32B / Qwen3-235B-A22B cost tables on the B200 GpuSpec), the
reference's partition, dispatch list digest, expected timeline/bubble,
stage feasibility and protocol edge digest, so tests/test_planner_golden.py
can check the product anywhere (the GPU box has no /root/reference).
"""
import ctypes
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2604_27085_b200.planner import Planner  # noqa: E402

CASES = [  # (model, seq, N, M, M_R, iterations)
    ("tiny", 256, 4, 4, 4, 3),
    ("tiny", 4096, 4, 4, 4, 3),
    ("qwen3-1.7b", 4096, 4, 8, 8, 5),
    ("qwen3-1.7b", 4096, 8, 16, 16, 7),
    ("qwen3-8b", 4096, 1, 16, 16, 3),
    ("qwen3-8b", 4096, 2, 8, 8, 5),
    ("qwen3-8b", 4096, 4, 8, 8, 7),
    ("qwen3-8b", 4096, 8, 16, 16, 7),
    ("qwen3-32b", 8192, 8, 16, 16, 7),
    ("qwen3-235b-a22b", 31744, 8, 16, 16, 5),
]


def digest(arr) -> str:
    return hashlib.sha256(arr.tobytes()).hexdigest()[:32]


def case_record(pl: Planner, cfg_src: Planner, model, seq, N, M, MR, iters):
    m = cfg_src.load_model(os.path.join(ROOT, "configs", "models", model + ".json"))
    g = cfg_src.load_gpu(os.path.join(ROOT, "configs", "gpus", "b200.json"))
    costs = pl.layer_costs(m, seq, 1, g, True)
    plan = pl.optimal_partition(costs, N, M)
    durs = pl.slot_durations(plan, costs)
    rec = {"model": model, "seq": seq, "N": N, "M": M, "M_R": MR, "iters": iters,
           "costs": costs.tolist(),
           "plan": {"fwd": [[r.first, r.last] for r in plan.fwd_stages],
                    "fused": [plan.fused_stage.first, plan.fused_stage.last],
                    "bwd": [[r.first, r.last] for r in plan.bwd_stages],
                    "t_max_ns": plan.t_max_ns, "objective": plan.objective},
           "slot_durs": durs}
    for kind, barrier in (("roundpipe-sync", True), ("roundpipe", False)):
        s = pl.synthesize(kind, N, M, MR, iters if kind == "roundpipe" else 1, durs)
        rep = pl.simulate(s, barrier)
        r = {"n_tasks": int(len(s.tasks)), "tasks_sha": digest(s.tasks),
             "timeline_sha": digest(rep.timeline), "makespan_ns": rep.makespan_ns,
             "bubble_num": rep.bubble_num, "bubble_den": rep.bubble_den,
             "first_tasks": s.tasks[:8].tolist()}
        if kind == "roundpipe" and iters >= 3:
            lo, hi = max(iters // 2 - 1, 1), min(iters // 2 + 1, iters - 2)
            r["interior"] = list(pl.interior_bubble(rep.timeline, N, lo, hi))
            r["interior_window"] = [lo, hi]
        rec[kind] = r
    rec["feasibility"] = [list(v) for v in pl.stage_feasibility(plan, costs, g, M)]
    L = len(costs)
    proto = pl.build_protocol(L, 2)
    rec["protocol"] = {"L": L, "T": 2, "n_actions": len(proto.actions),
                       "n_edges": len(proto.edges),
                       "edges_sha": hashlib.sha256(
                           json.dumps(proto.edges).encode()).hexdigest()[:32]}
    return rec


def main():
    ref = Planner(ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_planner.so")),
                  "ref_")
    out = {"generator": "tests/golden/make_planner_golden.py (reference planner)",
           "cases": [case_record(ref, ref, *c) for c in CASES],
           "protocol_makespans": {
               f"{L},{T},{mode}": ref.protocol_makespan(L, T, mode)
               for L, T in [(2, 2), (4, 3), (3, 4), (37, 2)]
               for mode in ("event-per-layer", "event-per-model", "blocking")}}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "planner_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
