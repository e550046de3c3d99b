"""Planner parity: product C-ABI vs the reference planner built from source.

The oracle (oracle/_ref/libref_planner.so) is the UNMODIFIED reference
header library (/root/reference/proj/include/roundpipe) behind the same ABI
glue; every output here must be bit-identical: stage plans, dispatch lists
(stage->GPU assignment and execution order), expected timelines, bubble
ratios, LPT placements, protocol action/edge lists, witnesses, makespans and
error codes. Seeds are fixed; instance sizes keep the suite to seconds.
"""
import random

import numpy as np
import pytest

from paper_2604_27085_b200 import _native
from paper_2604_27085_b200.planner import COST_DTYPE, INT64_MAX, Schedule


def rand_costs(rng, L, tmax=60, head=False, bwd_ratio=3):
    c = np.zeros(L, dtype=COST_DTYPE)
    for i in range(L):
        t = rng.randint(1, tmax)
        c[i] = (t, bwd_ratio * t if bwd_ratio else rng.randint(1, 3 * tmax),
                rng.randint(1, 1000), rng.randint(1, 100), rng.randint(1, 500))
    if head:
        c[-1]["t_fwd_ns"] *= 3
        c[-1]["t_bwd_ns"] *= 3
    return c


def outcome(fn, *a, **k):
    try:
        return ("ok", fn(*a, **k))
    except _native.NativeError as e:
        return ("err", e.code)


def test_candidate_tmax(product, oracle):
    rng = random.Random(11)
    for _ in range(40):
        c = rand_costs(rng, rng.randint(1, 25), bwd_ratio=rng.choice([0, 3]))
        assert product.candidate_tmax(c) == oracle.candidate_tmax(c)


@pytest.mark.parametrize("seed", range(6))
def test_optimal_partition_random(product, oracle, seed):
    rng = random.Random(1000 + seed)
    for trial in range(60):
        L = rng.randint(1, 40)
        c = rand_costs(rng, L, tmax=rng.choice([5, 60, 10**6]),
                       head=rng.random() < 0.5, bwd_ratio=rng.choice([0, 3, 3]))
        N = rng.randint(1, 8)
        M = N * rng.randint(1, 4) + rng.choice([0, 0, 1])
        total = int(c["param_bytes"].sum())
        mem = rng.choice([INT64_MAX, INT64_MAX, total, total // 3, 4 * total, 1])
        res = rng.choice([2.0, 1.0, 2.5])
        a = outcome(product.optimal_partition, c, N, M, mem, res)
        b = outcome(oracle.optimal_partition, c, N, M, mem, res)
        assert a == b, (trial, L, N, M, mem, res)


def test_partition_degenerate_inputs(product, oracle):
    c = rand_costs(random.Random(3), 5)
    for N, M in [(0, 1), (2, 1), (1, 0), (3, 2)]:
        assert outcome(product.optimal_partition, c, N, M) == \
            outcome(oracle.optimal_partition, c, N, M)
    empty = np.zeros(0, dtype=COST_DTYPE)
    assert outcome(product.optimal_partition, empty, 1, 1) == \
        outcome(oracle.optimal_partition, empty, 1, 1)
    # zero-duration layers (non-positive candidates are skipped)
    z = np.zeros(4, dtype=COST_DTYPE)
    z["param_bytes"] = 1
    assert outcome(product.optimal_partition, z, 1, 1) == \
        outcome(oracle.optimal_partition, z, 1, 1)


def test_greedy_pack_random(product, oracle):
    rng = random.Random(77)
    for _ in range(200):
        c = rand_costs(rng, rng.randint(1, 20))
        N = rng.randint(1, 4)
        M = N * rng.randint(1, 3)
        cands = oracle.candidate_tmax(c)
        t = rng.choice(cands + [1, max(cands) * 2])
        mem = rng.choice([INT64_MAX, int(c["param_bytes"].sum())])
        assert outcome(product.greedy_pack, c, N, M, t, mem) == \
            outcome(oracle.greedy_pack, c, N, M, t, mem)


def test_symmetric_split_random(product, oracle):
    rng = random.Random(5)
    for _ in range(100):
        L = rng.randint(1, 30)
        c = rand_costs(rng, L)
        S = rng.randint(0, L + 1)
        assert outcome(product.symmetric_split, c, S) == \
            outcome(oracle.symmetric_split, c, S)


def _same_schedule(a, b):
    assert a[0] == b[0]
    if a[0] == "err":
        assert a[1] == b[1]
        return
    sa, sb = a[1], b[1]
    assert (sa.num_gpus, sa.slots_per_iteration) == (sb.num_gpus, sb.slots_per_iteration)
    assert np.array_equal(sa.tasks, sb.tasks)


def test_synthesize_roundpipe_random(product, oracle):
    rng = random.Random(21)
    for _ in range(150):
        N = rng.randint(1, 8)
        S = rng.randint(1, 20)
        MR = rng.choice([0, N, 2 * N, N + 1, N - 1 if N > 1 else 1])
        M = rng.choice([N, 2 * N, 4 * N, 6 * N, 5 * N + 1])
        iters = rng.randint(1, 4)
        kind = rng.choice(["roundpipe", "roundpipe-sync"])
        durs = [rng.randint(1, 100) for _ in range(S)]
        _same_schedule(outcome(product.synthesize, kind, N, M, MR, iters, durs),
                       outcome(oracle.synthesize, kind, N, M, MR, iters, durs))


def test_synthesize_baselines_random(product, oracle):
    rng = random.Random(22)
    for _ in range(150):
        kind = rng.choice(["gpipe", "1f1b", "interleaved-1f1b", "looped-bfs"])
        N = rng.randint(1, 8)
        v = rng.randint(1, 3)
        S = N if kind in ("gpipe", "1f1b") else v * N + rng.choice([0, 0, 1])
        M = rng.randint(1, 4 * N)
        f = [rng.randint(1, 50) for _ in range(S)]
        b = [rng.randint(1, 150) for _ in range(S)]
        _same_schedule(
            outcome(product.synthesize, kind, N, M, 0, 1, (), f, b),
            outcome(oracle.synthesize, kind, N, M, 0, 1, (), f, b))


def test_default_round_rule(product, oracle):
    for M in range(1, 70):
        for N in range(1, 9):
            assert product.default_round_micro_batches(M, N) == \
                oracle.default_round_micro_batches(M, N)


def test_validate_mutations(product, oracle):
    rng = random.Random(9)
    for _ in range(120):
        N = rng.randint(1, 6)
        s = product.synthesize("roundpipe", N, 2 * N, 0, 2,
                               [rng.randint(1, 9) for _ in range(rng.randint(1, 8))])
        t = s.tasks.copy()
        m = rng.randint(0, 5)
        i, j = rng.randrange(len(t)), rng.randrange(len(t))
        if m == 0:
            t = np.concatenate([t, t[i:i + 1]])
        elif m == 1:
            t[[i, j]] = t[[j, i]]
        elif m == 2:
            t[i]["gpu"] = (t[i]["gpu"] + 1) % N
        elif m == 3:
            t[i]["dur_ns"] = 0
        elif m == 4:
            t[i]["slot"] = s.slots_per_iteration
        m2 = Schedule(s.kind, s.num_gpus, s.slots_per_iteration, t)
        assert (product.validate(m2) is None) == (oracle.validate(m2) is None)


def _same_report(a, b):
    assert a[0] == b[0]
    if a[0] == "err":
        assert a[1] == b[1]
        return
    ra, rb = a[1], b[1]
    for k in ("makespan_ns", "span_ns", "busy_total_ns", "busy_per_gpu_ns",
              "bubble_num", "bubble_den", "bubble_ratio"):
        assert getattr(ra, k) == getattr(rb, k), k
    assert np.array_equal(ra.timeline, rb.timeline)


def test_simulate_random(product, oracle):
    rng = random.Random(33)
    for _ in range(80):
        kind = rng.choice(["roundpipe", "roundpipe-sync", "gpipe", "1f1b",
                           "interleaved-1f1b", "looped-bfs"])
        N = rng.randint(1, 6)
        if kind.startswith("roundpipe"):
            S = rng.randint(1, 14)
            s = product.synthesize(kind, N, 2 * N, rng.choice([0, N]),
                                   rng.randint(1, 5),
                                   [rng.randint(1, 1000) for _ in range(S)])
        else:
            S = N if kind in ("gpipe", "1f1b") else 2 * N
            s = product.synthesize(kind, N, rng.randint(1, 3 * N), 0, 1, (),
                                   [rng.randint(1, 90) for _ in range(S)],
                                   [rng.randint(1, 250) for _ in range(S)])
        barrier = rng.random() < 0.5
        delay = rng.choice([0, 0, 7, 1000])
        _same_report(outcome(product.simulate, s, barrier, delay),
                     outcome(oracle.simulate, s, barrier, delay))


def test_simulate_deadlock_and_malformed(product, oracle):
    t = np.zeros(1, dtype=product.synthesize("gpipe", 1, 1, 0, 1, (), [1], [1]).tasks.dtype)
    t[0] = (0, 0, 1, 0, 0, 0, 10)
    s = Schedule("gpipe", 1, 2, t)
    assert outcome(product.simulate, s) == outcome(oracle.simulate, s) == ("err", 5)


def test_bubble_windows(product, oracle):
    rng = random.Random(44)
    for _ in range(40):
        N = rng.randint(1, 8)
        S = rng.randint(N, 3 * N)
        s = product.synthesize("roundpipe", N, 2 * N, 0, 7,
                               [rng.randint(100, 900) for _ in range(S)])
        rep = product.simulate(s)
        lo, hi = rng.randint(0, 3), rng.randint(3, 6)
        assert product.interior_bubble(rep.timeline, N, lo, hi) == \
            oracle.interior_bubble(rep.timeline, N, lo, hi)
        w0 = rng.randint(0, rep.makespan_ns // 2)
        w1 = w0 + rng.randint(1, rep.makespan_ns)
        assert product.idle_in_window(rep.timeline, N, w0, w1) == \
            oracle.idle_in_window(rep.timeline, N, w0, w1)


def test_transfer_plan_random(product, oracle):
    rng = random.Random(55)
    for _ in range(150):
        n = rng.randint(1, 14)
        items = [(f"t{rng.randint(0, 30)}", rng.randint(1, 1000), rng.randint(0, 1))
                 for _ in range(n)]
        ids = [i[0] for i in items]
        if len(set(ids)) != len(ids):  # duplicate ids are ambiguous under std::sort
            items = [(f"u{k}",) + i[1:] for k, i in enumerate(items)]
        M = rng.randint(1, 9)
        mc = rng.choice([0, 0, 1, 50, 10**9])
        a, b = outcome(product.plan, items, M, mc), outcome(oracle.plan, items, M, mc)
        assert a[0] == b[0]
        if a[0] == "ok":
            assert np.array_equal(a[1].chunks, b[1].chunks)
            assert a[1].window_totals == b[1].window_totals
            assert a[1].makespan_bytes == b[1].makespan_bytes
    for sizes, M in [([9, 7, 6, 5, 4], 3), ([1] * 12, 5), ([7], 3)]:
        assert product.optimal_makespan(sizes, M) == oracle.optimal_makespan(sizes, M)


def test_stage_feasibility_random(product, oracle):
    rng = random.Random(66)
    for _ in range(60):
        c = rand_costs(rng, rng.randint(2, 30), tmax=10**6)
        c["param_bytes"] *= 10**5
        c["act_ckpt_bytes"] *= 10**4
        N = rng.randint(1, 8)
        M = N * 2
        plan = oracle.optimal_partition(c, N, M)
        gpu = product.load_gpu("b200")
        gpu.link_bandwidth = rng.choice([32e9, 64e9, 1e6])
        assert product.stage_feasibility(plan, c, gpu, M) == \
            oracle.stage_feasibility(plan, c, gpu, M)


@pytest.mark.parametrize("mode", ["event-per-layer", "event-per-model", "blocking"])
def test_protocol_lists_and_checker(product, oracle, mode):
    for L in range(1, 5):
        for T in range(1, 4):
            for drop in range(0, 5):
                a = product.build_protocol(L, T, mode, drop)
                b = oracle.build_protocol(L, T, mode, drop)
                assert (a.actions, a.edges, a.gpu_actions) == \
                    (b.actions, b.edges, b.gpu_actions)
                assert product.check_all_interleavings(L, T, mode, drop) == \
                    oracle.check_all_interleavings(L, T, mode, drop)
                assert product.protocol_makespan(L, T, mode, drop) == \
                    oracle.protocol_makespan(L, T, mode, drop)


def test_protocol_runtime_sizes(product, oracle):
    # the executor instantiates EventPerLayer for L+1 = 37 (Qwen3-8B + head)
    for L, T in [(37, 2), (29, 3)]:
        a = product.build_protocol(L, T)
        b = oracle.build_protocol(L, T)
        assert (a.actions, a.edges) == (b.actions, b.edges)
        assert product.check_all_interleavings(L, T) == oracle.check_all_interleavings(L, T)
    assert outcome(product.check_all_interleavings, 3, 3, "event-per-layer", 0, 2) == \
        outcome(oracle.check_all_interleavings, 3, 3, "event-per-layer", 0, 2)
    dur = {"upload_ns": 5, "grad_write_ns": 7, "step_ns": 11, "p_copy_ns": 2,
           "g_copy_ns": 3}
    for mode in ("event-per-layer", "event-per-model", "blocking"):
        assert product.protocol_makespan(9, 4, mode, 0, dur) == \
            oracle.protocol_makespan(9, 4, mode, 0, dur)


def test_cost_tables_bundled_models(product, oracle):
    for model in ("qwen3-1.7b", "qwen3-32b", "qwen3-235b", "llama-3.1-8b", "gpt-oss-20b"):
        m = oracle.load_model(model)  # reference configs
        g = oracle.load_gpu("rtx4090")
        for s, b in [(2048, 4), (4096, 1), (31744, 1)]:
            for head in (False, True):
                assert np.array_equal(product.layer_costs(m, s, b, g, head),
                                      oracle.layer_costs(m, s, b, g, head))


def test_gantt_and_measured_report(product, oracle):
    """svg::render_gantt of simulated and 'measured' (jittered) timelines is
    byte-identical to the reference's; the measured-timeline report equals
    simulate()'s scalars on a simulated timeline (simulator.hpp:134-151)."""
    from paper_2604_27085_b200.planner import report_json
    rng = random.Random(55)
    for trial in range(12):
        N = rng.randint(1, 6)
        L = rng.randint(2, 12)
        c = rand_costs(rng, L + 1, head=True)
        M = N * rng.randint(1, 3)
        plan = product.optimal_partition(c, N, M)
        durs = product.slot_durations(plan, c)
        s = product.synthesize("roundpipe", N, M, 0, 3, durs)
        rep = product.simulate(s)
        tl = rep.timeline.copy()
        if trial % 2:  # measured timelines start late / stretch / shrink
            tl["start_ns"] += rng.randint(0, 50)
            tl["end_ns"] = tl["start_ns"] + (tl["dur_ns"] * rng.uniform(0.8, 1.3)).astype(np.int64)
        for p in (None, plan):
            a = product.render_gantt(tl, N, p, width=900)
            assert a == oracle.render_gantt(tl, N, p, width=900)
            assert a.startswith("<svg") and a.count("<rect") >= len(tl)
        mr = product.timeline_report(rep.timeline, N)
        assert (mr.makespan_ns, mr.span_ns, mr.busy_total_ns, mr.bubble_num, mr.bubble_den,
                mr.bubble_ratio, mr.busy_per_gpu_ns) == \
            (rep.makespan_ns, rep.span_ns, rep.busy_total_ns, rep.bubble_num, rep.bubble_den,
             rep.bubble_ratio, rep.busy_per_gpu_ns)
        j = report_json(mr, N)
        assert len(j["events"]) == len(tl) and j["bubble_den"] == N * j["span_ns"]
