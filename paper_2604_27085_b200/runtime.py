"""Python front-end of the RoundPipe runtime C-ABI (include/rp/runtime.h).

Mirrors the paper's user interface: ``forward_backward``
returns the loss as soon as it is known, ``step`` queues the optimizer,
``sync`` drains. Only host numpy buffers cross the ABI; all compute happens
in libroundpipe_b200.so (no fallback).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native
from .planner import EVENT_DTYPE, COST_DTYPE, LayerRange, StagePlan, RangeC, StagePlanC

I32, I64, F32, F64, VP = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_void_p
P = C.POINTER

RP_RT_SKIP_INIT = 1
RP_RT_RECORD_TIMELINE = 2
RP_RT_FUSED_PIPELINE = 4
RP_RT_UNFUSED_SWIGLU = 8
RP_RT_RECORD_PROTOCOL = 16
RP_RT_HOST_PUBLISH = 32
RP_RT_POOLED = 64


class AdamC(C.Structure):
    _fields_ = [("lr", F32), ("beta1", F32), ("beta2", F32), ("eps", F32),
                ("weight_decay", F32), ("grad_scale", F32)]


class RuntimeConfigC(C.Structure):
    _fields_ = [("model", C.c_char_p), ("seq_len", I32), ("micro_batch", I32),
                ("micro_batches", I32), ("round_micro_batches", I32), ("num_gpus", I32),
                ("async_optimizer", I32), ("mem_limit_bytes", I64), ("residency_factor", F64),
                ("costs", VP), ("n_costs", I32), ("adam", AdamC), ("init_seed", C.c_uint64),
                ("init_std", F32), ("flags", I32), ("lora_rank", I32), ("lora_alpha", F32),
                ("resident_state_gb", F64), ("logits_rows", I32), ("reserved_", I32)]


class StatsC(C.Structure):
    _fields_ = [("num_layers", I32), ("num_slots", I32), ("params_total", I64),
                ("host_bytes_pinned", I64), ("device_bytes", I64 * 8), ("h2d_bytes", I64),
                ("d2h_bytes", I64), ("p2p_bytes", I64), ("iterations_done", I32),
                ("kernels_launched", I32), ("pad_", I32), ("resident_params", I64),
                ("pool_peak_bytes", I64), ("pool_bytes", I64)]


LAYER_TENSORS = ["input_norm", "qkv", "q_norm", "k_norm", "o", "post_norm", "gate_up", "down"]
# Qwen3-MoE layers: router [E, h], experts stacked gate_up [E*2m, h], down [E*h, m]
MOE_LAYER_TENSORS = ["input_norm", "qkv", "q_norm", "k_norm", "o", "post_norm", "router",
                     "gate_up", "down"]
LORA_TENSORS = ["qkv_lora_A", "qkv_lora_B", "o_lora_A", "o_lora_B", "gate_up_lora_A",
                "gate_up_lora_B", "down_lora_A", "down_lora_B"]
HEAD_TENSORS = ["final_norm", "lm_head"]


class MemoryPlanC(C.Structure):
    _fields_ = [("num_slots", I32), ("pooled", I32), ("pool_worker", I32), ("pad_", I32),
                ("mem_limit_bytes", I64), ("activations", I64), ("scratch", I64),
                ("handoff", I64), ("optimizer_ring", I64), ("workspace", I64),
                ("static_groups", I64), ("pool_peak", I64), ("pool_weights", I64),
                ("pool_grads", I64), ("pool_pend", I64), ("pool_checkpoints", I64),
                ("total_static", I64), ("total_pooled", I64)]


def memory_plan(model="qwen3-8b", seq_len=4096, micro_batch=1, micro_batches=16, num_gpus=1,
                round_micro_batches=0, async_optimizer=True, hbm_bytes=int(180e9),
                lora_rank=0, pooled=False, mem_limit_bytes=0) -> dict:
    """Per-worker device-memory plan of a configuration, on the host (no GPU):
    rp_memory_plan (include/rp/runtime.h)."""
    lib = _native.load()
    name = model.encode()
    cfg = RuntimeConfigC(name, seq_len, micro_batch, micro_batches, round_micro_batches, num_gpus,
                         int(async_optimizer), mem_limit_bytes, 2.0, VP(0), 0,
                         AdamC(1e-4, 0.9, 0.95, 1e-8, 0.0, 1.0), 0, 0.02,
                         RP_RT_POOLED if pooled else 0, lora_rank, 0.0, -1.0, 0, 0)
    out = MemoryPlanC()
    f = lib.rp_memory_plan
    f.restype = C.c_int
    code = f(C.byref(cfg), I64(hbm_bytes), C.byref(out))
    if code != 0:
        raise _native._ERRORS.get(code, _native.NativeError)(code, "rp_memory_plan failed")
    return {k: getattr(out, k) for k, _ in MemoryPlanC._fields_ if k != "pad_"}


@dataclass
class AdamW:
    lr: float = 1e-4
    betas: tuple = (0.9, 0.95)
    eps: float = 1e-8
    weight_decay: float = 0.0


class RoundPipe:
    """One RoundPipe training runtime over N workers (logical GPUs mapped onto
    the visible B200s; N workers on one device run the full N-way dispatch)."""

    def __init__(self, model="qwen3-8b", seq_len=4096, micro_batch=1, micro_batches=16,
                 num_gpus=1, round_micro_batches=0, async_optimizer=True, adam=AdamW(),
                 costs=None, mem_limit_bytes=0, residency_factor=2.0, init_seed=0,
                 init_std=0.02, skip_init=False, record_timeline=False, lora_rank=0,
                 lora_alpha=0.0, resident_state_gb=-1.0, logits_rows=0, fused_pipeline=False,
                 unfused_swiglu=False, record_protocol=False, host_publish=False,
                 pooled=False):
        """resident_state_gb: fp32 AdamW state placement on a single device —
        < 0 keeps the groups that fit in free HBM resident (default), 0 keeps
        all of it in pinned host memory (host-offloaded Adam, BASELINE
        configs[2]), > 0 caps the resident part in GB. logits_rows: LM-head
        chunk rows (0 = 2048)."""
        self.lib = _native.load()
        self._costs = None
        if costs is not None:
            self._costs = np.ascontiguousarray(costs, dtype=COST_DTYPE)
        self._model = model.encode()
        cfg = RuntimeConfigC(
            self._model, seq_len, micro_batch, micro_batches, round_micro_batches, num_gpus,
            int(async_optimizer), mem_limit_bytes, residency_factor,
            VP(self._costs.ctypes.data) if self._costs is not None else VP(0),
            len(self._costs) if self._costs is not None else 0,
            AdamC(adam.lr, adam.betas[0], adam.betas[1], adam.eps, adam.weight_decay, 1.0),
            init_seed, init_std,
            (RP_RT_SKIP_INIT if skip_init else 0) | (RP_RT_RECORD_TIMELINE if record_timeline else 0)
            | (RP_RT_FUSED_PIPELINE if fused_pipeline else 0)
            | (RP_RT_UNFUSED_SWIGLU if unfused_swiglu else 0)
            | (RP_RT_RECORD_PROTOCOL if record_protocol else 0)
            | (RP_RT_HOST_PUBLISH if host_publish else 0)
            | (RP_RT_POOLED if pooled else 0),
            lora_rank, lora_alpha, float(resident_state_gb), int(logits_rows), 0)
        self.h = VP()
        self._call("rp_runtime_create", C.byref(cfg), C.byref(self.h))
        # MoE layers carry a router and adapt the attention projections only
        self.moe = len(self.layout(0)) in (len(MOE_LAYER_TENSORS), len(MOE_LAYER_TENSORS) + 4)
        if self.moe:
            self.layer_tensors = MOE_LAYER_TENSORS + (LORA_TENSORS[:4] if lora_rank else [])
        else:
            self.layer_tensors = LAYER_TENSORS + (LORA_TENSORS if lora_rank else [])
        self.seq_len, self.micro_batch, self.micro_batches = seq_len, micro_batch, micro_batches
        self.num_gpus = num_gpus

    def _call(self, name, *args):
        f = getattr(self.lib, name)
        f.restype = C.c_int
        code = f(*args)
        if code != 0:
            le = self.lib.rp_runtime_last_error
            le.restype = C.c_char_p
            raise _native._ERRORS.get(code, _native.NativeError)(code, le().decode())

    def close(self):
        if self.h:
            self._call("rp_runtime_destroy", self.h)
            self.h = VP()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plan ----------------------------------------------------------------------
    def plan(self) -> tuple[StagePlan, list]:
        cap = 4096
        fwd, bwd = (RangeC * cap)(), (RangeC * cap)()
        p = StagePlanC()
        p.fwd, p.bwd, p.cap = C.cast(fwd, P(RangeC)), C.cast(bwd, P(RangeC)), cap
        durs = np.zeros(cap, dtype=np.int64)
        n = I32()
        self._call("rp_runtime_plan", self.h, C.byref(p), durs.ctypes.data_as(P(I64)),
                   I32(cap), C.byref(n))
        plan = StagePlan([LayerRange(fwd[i].first, fwd[i].last) for i in range(p.num_fwd)],
                         LayerRange(p.fused.first, p.fused.last),
                         [LayerRange(bwd[i].first, bwd[i].last) for i in range(p.num_bwd)],
                         p.t_max_ns, p.objective)
        return plan, durs[: n.value].tolist()

    def costs(self) -> np.ndarray:
        out = np.zeros(4096, dtype=COST_DTYPE)
        n = I32()
        self._call("rp_runtime_costs", self.h, out.ctypes.data_as(VP), I32(len(out)), C.byref(n))
        return out[: n.value]

    def save(self, path: str):
        """Checkpoint the host state (fp32 master, Adam m/v, steps, bf16 master)."""
        self._call("rp_runtime_save", self.h, str(path).encode())

    def load(self, path: str):
        """Resume from rp_runtime_save's file (same model); device caches reset."""
        self._call("rp_runtime_load", self.h, str(path).encode())

    def measured_costs(self) -> np.ndarray:
        """Cost table measured on the profiled steps: per layer
        t_fwd / t_bwd (fwd+bwd) kernel ns of one micro-batch; bytes from the
        cost model. Pass as ``costs=`` to re-plan on measured costs."""
        out = np.zeros(4096, dtype=COST_DTYPE)
        n = I32()
        self._call("rp_runtime_measured_costs", self.h, out.ctypes.data_as(VP), I32(len(out)),
                   C.byref(n))
        return out[: n.value]

    # -- parameters --------------------------------------------------------------------
    def param_count(self, group: int) -> int:
        n = I64()
        self._call("rp_param_count", self.h, I32(group), C.byref(n))
        return n.value

    def layout(self, group: int):
        offs, rows, cols = (np.zeros(16, dtype=np.int64) for _ in range(3))
        n = I32()
        self._call("rp_param_layout", self.h, I32(group), offs.ctypes.data_as(P(I64)),
                   rows.ctypes.data_as(P(I64)), cols.ctypes.data_as(P(I64)), I32(16), C.byref(n))
        return [(int(offs[i]), int(rows[i]), int(cols[i])) for i in range(n.value)]

    def set_group(self, group: int, flat: np.ndarray):
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        self._call("rp_set_params", self.h, I32(group), flat.ctypes.data_as(P(F32)),
                   I64(flat.size))

    def get_group(self, group: int, which: int = 0) -> np.ndarray:
        out = np.zeros(self.param_count(group), dtype=np.float32)
        self._call("rp_get_params", self.h, I32(group), I32(which), out.ctypes.data_as(P(F32)),
                   I64(out.size))
        return out

    def load_state(self, params: dict, num_layers: int):
        """params: oracle-style dict name -> fp32 tensor/ndarray
        (embed, layers.{l}.<LAYER_TENSORS>, head.<HEAD_TENSORS>)."""
        def pack(group, names):
            flat = np.zeros(self.param_count(group), dtype=np.float32)
            for (off, r, c), name in zip(self.layout(group), names):
                v = np.asarray(params[name], dtype=np.float32).reshape(-1)
                assert v.size == r * c, (name, v.size, r, c)
                flat[off:off + v.size] = v
            self.set_group(group, flat)
        pack(-1, ["embed"])
        for l in range(num_layers):
            pack(l, [f"layers.{l}.{n}" for n in self.layer_tensors])
        pack(num_layers, [f"head.{n}" for n in HEAD_TENSORS])

    def read_state(self, num_layers: int, which: int = 0) -> dict:
        out = {}

        def unpack(group, names):
            flat = self.get_group(group, which)
            for (off, r, c), name in zip(self.layout(group), names):
                out[name] = flat[off:off + r * c].reshape((r, c) if c > 1 else (r,))
        unpack(-1, ["embed"])
        for l in range(num_layers):
            unpack(l, [f"layers.{l}.{n}" for n in self.layer_tensors])
        unpack(num_layers, [f"head.{n}" for n in HEAD_TENSORS])
        return out

    # -- training ----------------------------------------------------------------------
    def forward_backward(self, tokens: np.ndarray, labels: np.ndarray) -> float:
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        n = self.micro_batches * self.micro_batch * self.seq_len
        if tokens.size != n or labels.size != n:
            raise ValueError(f"tokens/labels need {n} entries ([M, b, s]), got "
                             f"{tokens.size} / {labels.size}")
        loss = F32()
        self._call("rp_forward_backward", self.h, tokens.ctypes.data_as(P(I32)),
                   labels.ctypes.data_as(P(I32)), C.byref(loss))
        return loss.value

    def forward_backward_async(self, tokens: np.ndarray, labels: np.ndarray) -> int:
        """Enqueue the iteration and return its index without waiting; the
        host buffers may be reused at once. Read the loss with loss(it)."""
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        n = self.micro_batches * self.micro_batch * self.seq_len
        if tokens.size != n or labels.size != n:
            raise ValueError(f"tokens/labels need {n} entries ([M, b, s]), got "
                             f"{tokens.size} / {labels.size}")
        it = I32()
        self._call("rp_forward_backward_async", self.h, tokens.ctypes.data_as(P(I32)),
                   labels.ctypes.data_as(P(I32)), C.byref(it))
        return it.value

    def loss(self, iteration: int) -> float:
        """Mean token loss of one of the two most recently enqueued iterations."""
        out = F32()
        self._call("rp_loss", self.h, I32(iteration), C.byref(out))
        return out.value

    def step(self):
        self._call("rp_step", self.h)

    def sync(self):
        self._call("rp_sync", self.h)

    def timeline(self) -> np.ndarray:
        cap = 1 << 20
        ev = np.zeros(cap, dtype=EVENT_DTYPE)
        n = I64()
        self._call("rp_timeline", self.h, ev.ctypes.data_as(VP), I64(cap), C.byref(n))
        return ev[: n.value].copy()

    def clear_timeline(self):
        self._call("rp_timeline_clear", self.h)

    PROTO_DTYPE = np.dtype([("before_kind", "<i4"), ("before_group", "<i4"),
                            ("before_iteration", "<i4"), ("after_kind", "<i4"),
                            ("after_group", "<i4"), ("after_iteration", "<i4")])

    def protocol_edges(self) -> np.ndarray:
        """Realised hand-off edges (record_protocol=True): (kind, group,
        iteration) waited on -> waiting; kinds as consistency.hpp ActionKind."""
        cap = 1 << 20
        ev = np.zeros(cap, dtype=self.PROTO_DTYPE)
        n = I64()
        self._call("rp_runtime_protocol_edges", self.h, ev.ctypes.data_as(VP), I64(cap), C.byref(n))
        return ev[: n.value].copy()

    def progress(self, group: int = -1) -> tuple:
        """(latest p_copy index published for `group`, latest iteration whose
        loss is on the host), read from the host-mapped flag words."""
        pub, it = I32(), I32()
        self._call("rp_runtime_progress", self.h, I32(group), C.byref(pub), C.byref(it))
        return pub.value, it.value

    XFER_DTYPE = np.dtype([("kind", "<i4"), ("group", "<i4"), ("iteration", "<i4"),
                           ("worker", "<i4"), ("start_ns", "<i8"), ("end_ns", "<i8")])

    def transfer_timeline(self) -> np.ndarray:
        """kind 0 = weight upload, 1 = p_copy, 2 = AdamW over a group."""
        cap = 1 << 18
        ev = np.zeros(cap, dtype=self.XFER_DTYPE)
        n = I64()
        self._call("rp_transfer_timeline", self.h, ev.ctypes.data_as(VP), I64(cap), C.byref(n))
        return ev[: n.value].copy()

    def stats(self) -> dict:
        st = StatsC()
        self._call("rp_runtime_stats", self.h, C.byref(st))
        return {"num_layers": st.num_layers, "num_slots": st.num_slots,
                "params_total": st.params_total, "host_bytes_pinned": st.host_bytes_pinned,
                "device_bytes": list(st.device_bytes), "h2d_bytes": st.h2d_bytes,
                "d2h_bytes": st.d2h_bytes, "p2p_bytes": st.p2p_bytes,
                "iterations_done": st.iterations_done, "kernels_launched": st.kernels_launched,
                "resident_params": st.resident_params, "pool_peak_bytes": st.pool_peak_bytes,
                "pool_bytes": st.pool_bytes}

    # -- profiling ----------------------------------------------------------------
    PROFILE_CATEGORIES = ("gemm", "attention", "hbm_kernels", "adamw")

    def profile(self, enable: bool):
        self._call("rp_runtime_profile", self.h, I32(int(enable)))

    def profile_read(self) -> dict:
        t = (C.c_double * 4)()
        w = (C.c_double * 4)()
        n = (I64 * 4)()
        self._call("rp_runtime_profile_read", self.h, t, w, n)
        return {c: {"ms": t[i], "work": w[i], "launches": n[i]}
                for i, c in enumerate(self.PROFILE_CATEGORIES)}

    PROF_DTYPE = np.dtype([("cat", "<i4"), ("worker", "<i4"), ("lane", "<i4"), ("pad", "<i4"),
                           ("start_ns", "<i8"), ("end_ns", "<i8"), ("work", "<f8")])

    def profile_records(self) -> np.ndarray:
        """Per-launch (category, worker, lane, start_ns, end_ns, work) of the
        profiled steps; lane 0 = compute stream, 1 = optimizer stream."""
        n = I64()
        cap = 1 << 20
        rec = np.zeros(cap, dtype=self.PROF_DTYPE)
        self._call("rp_runtime_profile_records", self.h, rec.ctypes.data_as(VP), I64(cap),
                   C.byref(n))
        return rec[: n.value].copy()
