"""Python mirror of the reference planner API over the product C-ABI.

Same names and argument meaning as the reference's C++ API
(proj/include/roundpipe/*.hpp) — ``optimal_partition``, ``synthesize``,
``simulate``, ``interior_bubble``, ``plan`` (LPT), ``build_protocol``,
``check_all_interleavings`` … — and the same error behaviour (exceptions
carrying the CLI exit-code taxonomy, proj/tools/roundpipe.cpp:25-29).

``Planner(lib, prefix)`` binds any library exporting the ABI; the product is
``Planner()``; the test suite also binds the reference build
(oracle/_ref/libref_planner.so, prefix ``ref_``) through the same class, so
parity tests call both sides with identical marshalling.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native

I32, I64, F64 = C.c_int32, C.c_int64, C.c_double
P = C.POINTER

# ---- ABI structs (include/rp/cabi.h) ---------------------------------------


class ModelConfigC(C.Structure):
    _fields_ = [("hidden_dim", F64), ("num_heads", I32), ("num_kv_heads", I32),
                ("intermediate_dim", F64), ("active_experts", I32),
                ("total_experts", I32), ("num_layers", I32), ("has_head", I32),
                ("head_flops_per_token", F64), ("has_head_param_bytes", I32),
                ("head_param_bytes", F64)]


class GpuSpecC(C.Structure):
    _fields_ = [("peak_fp16_flops", F64), ("memory_bytes", F64),
                ("link_bandwidth", F64)]


class LayerCostC(C.Structure):
    _fields_ = [("t_fwd_ns", I64), ("t_bwd_ns", I64), ("param_bytes", I64),
                ("act_ckpt_bytes", I64), ("act_full_bytes", I64)]


class RangeC(C.Structure):
    _fields_ = [("first", I32), ("last", I32)]


class StagePlanC(C.Structure):
    _fields_ = [("num_fwd", I32), ("num_bwd", I32), ("fused", RangeC),
                ("t_max_ns", I64), ("objective", I64), ("fwd", P(RangeC)),
                ("bwd", P(RangeC)), ("cap", I32)]


class SimReportC(C.Structure):
    _fields_ = [("makespan_ns", I64), ("span_ns", I64), ("busy_total_ns", I64),
                ("bubble_num", I64), ("bubble_den", I64), ("bubble_ratio", F64)]


class TransferChunkC(C.Structure):
    _fields_ = [("item", I32), ("chunk_index", I32), ("window", I32),
                ("position", I32), ("bytes", I64)]


class WindowVerdictC(C.Structure):
    _fields_ = [("slot", I32), ("feasible", I32), ("window_ns", I64),
                ("weight_bytes", I64), ("activation_bytes", I64)]


class ActionC(C.Structure):
    _fields_ = [("kind", I32), ("layer", I32), ("iteration", I32)]


class EdgeC(C.Structure):
    _fields_ = [("before", I32), ("after", I32)]


class DurationsC(C.Structure):
    _fields_ = [("upload_ns", I64), ("grad_write_ns", I64), ("step_ns", I64),
                ("p_copy_ns", I64), ("g_copy_ns", I64)]


TASK_DTYPE = np.dtype([("iteration", "<i4"), ("round", "<i4"), ("slot", "<i4"),
                       ("mb", "<i4"), ("gpu", "<i4"), ("pad_", "<i4"),
                       ("dur_ns", "<i8")])
EVENT_DTYPE = np.dtype([("iteration", "<i4"), ("round", "<i4"), ("slot", "<i4"),
                        ("mb", "<i4"), ("gpu", "<i4"), ("pad_", "<i4"),
                        ("dur_ns", "<i8"), ("start_ns", "<i8"), ("end_ns", "<i8")])
COST_DTYPE = np.dtype([("t_fwd_ns", "<i8"), ("t_bwd_ns", "<i8"),
                       ("param_bytes", "<i8"), ("act_ckpt_bytes", "<i8"),
                       ("act_full_bytes", "<i8")])

# enums (include/rp/cabi.h)
SCHEDULE_KINDS = {"roundpipe": 0, "roundpipe-sync": 1, "gpipe": 2, "1f1b": 3,
                  "interleaved-1f1b": 4, "looped-bfs": 5}
PROTOCOL_MODES = {"blocking": 0, "event-per-model": 1, "event-per-layer": 2}
ACTION_KINDS = ["param_upload", "grad_write", "opt_step", "p_copy", "g_copy"]
INT64_MAX = (1 << 63) - 1

# ---- value types ------------------------------------------------------------


@dataclass(frozen=True)
class LayerRange:
    first: int
    last: int

    def size(self) -> int:
        return 0 if self.last < self.first else self.last - self.first + 1


@dataclass
class StagePlan:
    fwd_stages: list
    fused_stage: LayerRange
    bwd_stages: list
    t_max_ns: int
    objective: int

    def num_slots(self) -> int:
        return len(self.fwd_stages) + 1 + len(self.bwd_stages)

    def slots(self):
        """(kind, LayerRange) in slot order: fwd…, fused, bwd… (scheduler.hpp:104)."""
        return ([("fwd", r) for r in self.fwd_stages] + [("fused", self.fused_stage)]
                + [("bwd", r) for r in self.bwd_stages])


@dataclass
class Schedule:
    kind: str
    num_gpus: int
    slots_per_iteration: int
    tasks: np.ndarray  # TASK_DTYPE, emission order


@dataclass
class SimReport:
    makespan_ns: int
    span_ns: int
    busy_total_ns: int
    busy_per_gpu_ns: list
    bubble_num: int
    bubble_den: int
    bubble_ratio: float
    timeline: np.ndarray  # EVENT_DTYPE, emission order


@dataclass
class TransferPlan:
    chunks: np.ndarray        # (item, chunk_index, window, position, bytes)
    window_totals: list
    makespan_bytes: int


@dataclass
class Protocol:
    layers: int
    iterations: int
    mode: str
    actions: list             # (kind, layer, iteration)
    gpu_actions: int
    edges: list               # (before, after)


@dataclass
class Verdict:
    ok: bool
    violated_constraint: int = 0
    witness: list = field(default_factory=list)


def costs_array(costs) -> np.ndarray:
    """Accept a COST_DTYPE array, a list of dicts/tuples, or LayerCostC list."""
    if isinstance(costs, np.ndarray) and costs.dtype == COST_DTYPE:
        return np.ascontiguousarray(costs)
    out = np.zeros(len(costs), dtype=COST_DTYPE)
    for i, c in enumerate(costs):
        if isinstance(c, dict):
            for k in COST_DTYPE.names:
                out[i][k] = c.get(k, 0)
        else:
            out[i] = tuple(c) + (0,) * (5 - len(tuple(c)))
    return out


class Planner:
    """Bindings for one library exporting the planner ABI under ``prefix``."""

    def __init__(self, lib: Optional[C.CDLL] = None, prefix: str = "rp_"):
        self.lib = lib if lib is not None else _native.load()
        self.p = prefix

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _call(self, name, *args):
        f = self._f(name)
        f.restype = C.c_int
        return _native.check(self.lib, self.p, f(*args))

    # -- cost model / config ---------------------------------------------------
    def load_model(self, name_or_path: str) -> ModelConfigC:
        m = ModelConfigC()
        self._call("load_model", name_or_path.encode(), C.byref(m))
        return m

    def load_gpu(self, name_or_path: str) -> GpuSpecC:
        g = GpuSpecC()
        self._call("load_gpu", name_or_path.encode(), C.byref(g))
        return g

    def layer_costs(self, cfg: ModelConfigC, seq_len: int, micro_batch: int,
                    gpu: GpuSpecC, include_head: bool = False) -> np.ndarray:
        cap = cfg.num_layers + 1
        out = np.zeros(cap, dtype=COST_DTYPE)
        n = I32()
        self._call("layer_costs", C.byref(cfg), I32(seq_len), I32(micro_batch),
                   C.byref(gpu), I32(int(include_head)),
                   out.ctypes.data_as(P(LayerCostC)), I32(cap), C.byref(n))
        return out[: n.value]

    # -- partitioner -----------------------------------------------------------
    def candidate_tmax(self, costs) -> list:
        c = costs_array(costs)
        n = I64()
        self._call_sized("candidate_tmax", c, n)
        out = np.zeros(n.value, dtype=np.int64)
        self._call("candidate_tmax", c.ctypes.data_as(P(LayerCostC)), I32(len(c)),
                   out.ctypes.data_as(P(I64)), I64(len(out)), C.byref(n))
        return out.tolist()

    def _call_sized(self, name, c, n):
        f = self._f(name)
        f.restype = C.c_int
        f(c.ctypes.data_as(P(LayerCostC)), I32(len(c)), None, I64(0), C.byref(n))

    @staticmethod
    def _plan_buf(L):
        fwd = (RangeC * max(L, 1))()
        bwd = (RangeC * max(L, 1))()
        p = StagePlanC()
        p.fwd = C.cast(fwd, P(RangeC))
        p.bwd = C.cast(bwd, P(RangeC))
        p.cap = max(L, 1)
        return p, (fwd, bwd)

    @staticmethod
    def _plan_from(p: StagePlanC) -> StagePlan:
        return StagePlan(
            [LayerRange(p.fwd[i].first, p.fwd[i].last) for i in range(p.num_fwd)],
            LayerRange(p.fused.first, p.fused.last),
            [LayerRange(p.bwd[i].first, p.bwd[i].last) for i in range(p.num_bwd)],
            p.t_max_ns, p.objective)

    @staticmethod
    def _plan_to(plan: StagePlan):
        L = max(len(plan.fwd_stages), len(plan.bwd_stages), 1)
        p, keep = Planner._plan_buf(L)
        p.num_fwd, p.num_bwd = len(plan.fwd_stages), len(plan.bwd_stages)
        for i, r in enumerate(plan.fwd_stages):
            p.fwd[i] = RangeC(r.first, r.last)
        for i, r in enumerate(plan.bwd_stages):
            p.bwd[i] = RangeC(r.first, r.last)
        p.fused = RangeC(plan.fused_stage.first, plan.fused_stage.last)
        p.t_max_ns, p.objective = plan.t_max_ns, plan.objective
        return p, keep

    def optimal_partition(self, costs, num_gpus: int, micro_batches: int,
                          mem_limit_bytes: int = INT64_MAX,
                          residency_factor: float = 2.0) -> StagePlan:
        c = costs_array(costs)
        p, keep = self._plan_buf(len(c))
        self._call("partition", c.ctypes.data_as(P(LayerCostC)), I32(len(c)),
                   I32(num_gpus), I32(micro_batches), I64(mem_limit_bytes),
                   F64(residency_factor), C.byref(p))
        return self._plan_from(p)

    def greedy_pack(self, costs, num_gpus, micro_batches, t_max,
                    mem_limit_bytes=INT64_MAX, residency_factor=2.0):
        c = costs_array(costs)
        p, keep = self._plan_buf(len(c))
        found = I32()
        self._call("greedy_pack", c.ctypes.data_as(P(LayerCostC)), I32(len(c)),
                   I32(num_gpus), I32(micro_batches), I64(mem_limit_bytes),
                   F64(residency_factor), I64(t_max), C.byref(p), C.byref(found))
        return self._plan_from(p) if found.value else None

    def symmetric_split(self, costs, num_stages: int) -> list:
        c = costs_array(costs)
        out = (RangeC * max(len(c), 1))()
        n = I32()
        self._call("symmetric_split", c.ctypes.data_as(P(LayerCostC)), I32(len(c)),
                   I32(num_stages), out, I32(len(out)), C.byref(n))
        return [LayerRange(out[i].first, out[i].last) for i in range(n.value)]

    def slot_durations(self, plan: StagePlan, costs) -> list:
        c = costs_array(costs)
        p, keep = self._plan_to(plan)
        out = np.zeros(plan.num_slots(), dtype=np.int64)
        n = I32()
        self._call("slot_durations", C.byref(p), c.ctypes.data_as(P(LayerCostC)),
                   I32(len(c)), out.ctypes.data_as(P(I64)), I32(len(out)), C.byref(n))
        return out[: n.value].tolist()

    # -- scheduler ---------------------------------------------------------------
    def default_round_micro_batches(self, M: int, N: int) -> int:
        f = self._f("default_round_micro_batches")
        f.restype = I32
        return f(I32(M), I32(N))

    def synthesize(self, kind: str, num_gpus: int, micro_batches: int,
                   round_micro_batches: int = 0, iterations: int = 1,
                   slot_durs: Sequence[int] = (),
                   stage_fwd_durs: Sequence[int] = (),
                   stage_bwd_durs: Sequence[int] = ()) -> Schedule:
        sd = np.asarray(slot_durs, dtype=np.int64)
        fd = np.asarray(stage_fwd_durs, dtype=np.int64)
        bd = np.asarray(stage_bwd_durs, dtype=np.int64)
        if len(fd) != len(bd):
            raise ValueError("stage_fwd_durs and stage_bwd_durs differ in length")
        n, ng, spi = I64(), I32(), I32()
        args = lambda out, cap: (  # noqa: E731
            I32(SCHEDULE_KINDS[kind]), I32(num_gpus), I32(micro_batches),
            I32(round_micro_batches), I32(iterations),
            sd.ctypes.data_as(P(I64)) if len(sd) else None, I32(len(sd)),
            fd.ctypes.data_as(P(I64)) if len(fd) else None,
            bd.ctypes.data_as(P(I64)) if len(bd) else None, I32(len(fd)),
            out, I64(cap), C.byref(n), C.byref(ng), C.byref(spi))
        f = self._f("synthesize")
        f.restype = C.c_int
        code = f(*args(None, 0))
        if code not in (0, 7):
            _native.check(self.lib, self.p, code)
        tasks = np.zeros(n.value, dtype=TASK_DTYPE)
        self._call("synthesize", *args(tasks.ctypes.data_as(C.c_void_p), len(tasks)))
        return Schedule(kind, ng.value, spi.value, tasks)

    def validate(self, sched: Schedule) -> Optional[str]:
        t = np.ascontiguousarray(sched.tasks, dtype=TASK_DTYPE)
        f = self._f("validate_schedule")
        f.restype = C.c_int
        code = f(I32(SCHEDULE_KINDS[sched.kind]), I32(sched.num_gpus),
                 I32(sched.slots_per_iteration), t.ctypes.data_as(C.c_void_p),
                 I64(len(t)))
        if code == 0:
            return None
        le = self._f("last_error")
        le.restype = C.c_char_p
        if code == 2:
            return le().decode()
        _native.check(self.lib, self.p, code)

    # -- simulator ---------------------------------------------------------------
    def simulate(self, sched: Schedule, barrier_between_iterations: bool = False,
                 optimizer_delay_ns: int = 0) -> SimReport:
        t = np.ascontiguousarray(sched.tasks, dtype=TASK_DTYPE)
        rep = SimReportC()
        busy = np.zeros(max(sched.num_gpus, 1), dtype=np.int64)
        ev = np.zeros(len(t), dtype=EVENT_DTYPE)
        self._call("simulate", I32(SCHEDULE_KINDS[sched.kind]), I32(sched.num_gpus),
                   I32(sched.slots_per_iteration), t.ctypes.data_as(C.c_void_p),
                   I64(len(t)), I32(int(barrier_between_iterations)),
                   I64(optimizer_delay_ns), C.byref(rep), busy.ctypes.data_as(P(I64)),
                   ev.ctypes.data_as(C.c_void_p))
        return SimReport(rep.makespan_ns, rep.span_ns, rep.busy_total_ns,
                         busy[: sched.num_gpus].tolist(), rep.bubble_num,
                         rep.bubble_den, rep.bubble_ratio, ev)

    def idle_in_window(self, timeline: np.ndarray, num_gpus: int, w0: int, w1: int):
        ev = np.ascontiguousarray(timeline, dtype=EVENT_DTYPE)
        num, den, r = I64(), I64(), F64()
        self._call("idle_in_window", ev.ctypes.data_as(C.c_void_p), I64(len(ev)),
                   I32(num_gpus), I64(w0), I64(w1), C.byref(num), C.byref(den),
                   C.byref(r))
        return r.value, num.value, den.value

    def interior_bubble(self, timeline: np.ndarray, num_gpus: int, iter_lo: int,
                        iter_hi: int):
        ev = np.ascontiguousarray(timeline, dtype=EVENT_DTYPE)
        num, den, r = I64(), I64(), F64()
        self._call("interior_bubble", ev.ctypes.data_as(C.c_void_p), I64(len(ev)),
                   I32(num_gpus), I32(iter_lo), I32(iter_hi), C.byref(num),
                   C.byref(den), C.byref(r))
        return r.value, num.value, den.value

    # -- reporting (measured or simulated timelines) -------------------------------
    def timeline_report(self, timeline: np.ndarray, num_gpus: int) -> SimReport:
        """SimReport scalars over a measured timeline (simulator.hpp:134-151)."""
        ev = np.ascontiguousarray(timeline, dtype=EVENT_DTYPE)
        rep = SimReportC()
        busy = np.zeros(num_gpus, dtype=np.int64)
        self._call("timeline_report", ev.ctypes.data_as(C.c_void_p), I64(len(ev)),
                   I32(num_gpus), C.byref(rep), busy.ctypes.data_as(P(I64)))
        return SimReport(rep.makespan_ns, rep.span_ns, rep.busy_total_ns, busy.tolist(),
                         rep.bubble_num, rep.bubble_den, rep.bubble_ratio, ev)

    def render_gantt(self, timeline: np.ndarray, num_gpus: int,
                     plan: Optional[StagePlan] = None, width: int = 1200) -> str:
        """svg::render_gantt (svg.hpp:26): one lane per GPU, colour per slot."""
        ev = np.ascontiguousarray(timeline, dtype=EVENT_DTYPE)
        sl = plan.slots() if plan is not None else []
        kinds = np.asarray([{"fwd": 0, "fused": 1, "bwd": 2}[k] for k, _ in sl] or [0],
                           dtype=np.int32)
        rng = (RangeC * max(len(sl), 1))(*[RangeC(r.first, r.last) for _, r in sl])
        n = I64()
        args = (ev.ctypes.data_as(C.c_void_p), I64(len(ev)), I32(num_gpus),
                kinds.ctypes.data_as(P(I32)), rng, I32(len(sl)), I32(width))
        self._call("render_gantt", *args, None, I64(0), C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        self._call("render_gantt", *args, buf, I64(n.value + 1), C.byref(n))
        return buf.value.decode()


    # -- transfer planner --------------------------------------------------------
    def plan(self, items: Sequence[tuple], num_windows: int,
             max_chunk_bytes: int = 0) -> TransferPlan:
        """items: (tensor_id, bytes[, direction 0=up/1=down])."""
        ids = (C.c_char_p * max(len(items), 1))(*[str(i[0]).encode() for i in items])
        byts = np.asarray([i[1] for i in items], dtype=np.int64)
        dirs = np.asarray([i[2] if len(i) > 2 else 0 for i in items], dtype=np.int32)
        n, mk = I64(), I64()
        totals = np.zeros(max(num_windows, 1), dtype=np.int64)
        f = self._f("transfer_plan")
        f.restype = C.c_int
        call = lambda out, cap: f(  # noqa: E731
            ids, byts.ctypes.data_as(P(I64)), dirs.ctypes.data_as(P(I32)),
            I32(len(items)), I32(num_windows), I64(max_chunk_bytes), out, I64(cap),
            C.byref(n), totals.ctypes.data_as(P(I64)), C.byref(mk))
        code = call(None, 0)
        if code not in (0, 7):
            _native.check(self.lib, self.p, code)
        chunks = (TransferChunkC * max(n.value, 1))()
        _native.check(self.lib, self.p, call(chunks, n.value))
        arr = np.array([(c.item, c.chunk_index, c.window, c.position, c.bytes)
                        for c in chunks[: n.value]], dtype=np.int64).reshape(-1, 5)
        return TransferPlan(arr, totals[:num_windows].tolist(), mk.value)

    def optimal_makespan(self, chunks: Sequence[int], num_windows: int) -> int:
        a = np.asarray(chunks, dtype=np.int64)
        out = I64()
        self._call("optimal_makespan", a.ctypes.data_as(P(I64)), I32(len(a)),
                   I32(num_windows), C.byref(out))
        return out.value

    def stage_feasibility(self, plan: StagePlan, costs, gpu: GpuSpecC,
                          micro_batches: int) -> list:
        c = costs_array(costs)
        p, keep = self._plan_to(plan)
        out = (WindowVerdictC * plan.num_slots())()
        n = I32()
        self._call("stage_feasibility", C.byref(p), c.ctypes.data_as(P(LayerCostC)),
                   I32(len(c)), C.byref(gpu), I32(micro_batches), out,
                   I32(len(out)), C.byref(n))
        return [(v.slot, bool(v.feasible), v.window_ns, v.weight_bytes,
                 v.activation_bytes) for v in out[: n.value]]

    # -- consistency ---------------------------------------------------------------
    def build_protocol(self, layers: int, iterations: int,
                       mode: str = "event-per-layer", drop_edge: int = 0) -> Protocol:
        na, ne, ga = I64(), I64(), I32()
        f = self._f("build_protocol")
        f.restype = C.c_int
        m = PROTOCOL_MODES[mode]
        code = f(I32(layers), I32(iterations), I32(m), I32(drop_edge), None, I64(0),
                 C.byref(na), C.byref(ga), None, I64(0), C.byref(ne))
        if code not in (0, 7):
            _native.check(self.lib, self.p, code)
        acts = (ActionC * max(na.value, 1))()
        edges = (EdgeC * max(ne.value, 1))()
        self._call("build_protocol", I32(layers), I32(iterations), I32(m),
                   I32(drop_edge), acts, I64(na.value), C.byref(na), C.byref(ga),
                   edges, I64(ne.value), C.byref(ne))
        return Protocol(layers, iterations, mode,
                        [(a.kind, a.layer, a.iteration) for a in acts[: na.value]],
                        ga.value, [(e.before, e.after) for e in edges[: ne.value]])

    def check_all_interleavings(self, layers: int, iterations: int,
                                mode: str = "event-per-layer", drop_edge: int = 0,
                                max_states: int = 1 << 24) -> Verdict:
        ok, viol, n = I32(), I32(), I64()
        cap = 4 * layers * iterations + iterations + 1
        wit = (ActionC * cap)()
        f = self._f("check_protocol")
        f.restype = C.c_int
        code = f(I32(layers), I32(iterations), I32(PROTOCOL_MODES[mode]),
                 I32(drop_edge), I64(max_states), C.byref(ok), C.byref(viol), wit,
                 I64(cap), C.byref(n))
        if code not in (0, 4):
            _native.check(self.lib, self.p, code)
        return Verdict(bool(ok.value), viol.value,
                       [(a.kind, a.layer, a.iteration) for a in wit[: n.value]])

    def protocol_makespan(self, layers: int, iterations: int,
                          mode: str = "event-per-layer", drop_edge: int = 0,
                          durations: Optional[dict] = None) -> int:
        d = DurationsC(2, 2, 3, 1, 1)
        for k, v in (durations or {}).items():
            setattr(d, k, v)
        out = I64()
        self._call("protocol_makespan", I32(layers), I32(iterations),
                   I32(PROTOCOL_MODES[mode]), I32(drop_edge), C.byref(d), C.byref(out))
        return out.value


def planner() -> Planner:
    return Planner()


def report_json(rep: SimReport, num_gpus: int) -> dict:
    """The reference CLI's report schema (proj/tools/roundpipe.cpp:70-90) for a
    simulated or measured SimReport."""
    tl = rep.timeline
    return {
        "makespan_ns": int(rep.makespan_ns), "span_ns": int(rep.span_ns),
        "bubble_ratio": float(rep.bubble_ratio), "bubble_num": int(rep.bubble_num),
        "bubble_den": int(rep.bubble_den),
        "gpus": [{"id": g, "busy_ns": int(rep.busy_per_gpu_ns[g])} for g in range(num_gpus)],
        "events": [{"iter": int(e["iteration"]), "round": int(e["round"]),
                    "slot": int(e["slot"]), "mb": int(e["mb"]), "gpu": int(e["gpu"]),
                    "start_ns": int(e["start_ns"]), "end_ns": int(e["end_ns"])} for e in tl],
    }
