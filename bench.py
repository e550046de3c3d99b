"""Benchmark: RoundPipe fine-tune step throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload = BASELINE configs[2], the metric's config: Qwen3-8B full fine-tune,
seq 4096, b=1, M=16 micro-batches per step (65,536 tokens), RoundPipe-async
(staleness-1 optimizer), fp32 AdamW master weights + m + v HOST-OFFLOADED in
pinned memory and streamed through the GPU every step (chunked H2D ->
fused AdamW kernel -> D2H), activation recompute wherever the reference
partitioner places backward stages (at N=1 it plans a single fused stage,
so nothing is recomputed). Synthetic seeded token ids, random-init weights.

One JSON line (rank 0):
* `value`: tokens/s over exactly K steps bracketed by full device
  synchronisation + CUDA events; the runtime is a single controller, rank 0
  drives all N workers (the other ranks wait at a barrier), so the max over
  ranks is rank 0's time. Includes the last step's optimizer drain.
* `e2e`: the same K steps through the public API by the host clock (token /
  label host buffers in, the loss read back every step).
* `roofline`: the dominant kernel family (tcgen05 GEMMs) inside one profiled
  step vs the measured sustained bf16 peak; `step_roofline`: the slower of
  executed FLOPs at that peak and streamed host-link bytes at the measured
  PCIe rates.
* `bubble`: the reference's interior_bubble (async) / idle_in_window (sync)
  on the MEASURED per-task timeline, next to the simulator's for the plan.
* `variants`: shorter labelled runs of the HBM-resident optimizer placement
  and of RoundPipe-sync on the same workload (not the headline).
* `cpu_baseline`: the fp32 CPU oracle (port) timed on a bounded sample of the
  same step on all host cores (see cpu_step_sample).
--impl reference times that CPU implementation alone (the reference has no
data-plane code), plus the reference's own control path
(oracle/_ref: partition + synthesize + simulate, single-threaded) and the C1
step end to end on the CPU oracle.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

def model_dims(model):
    """Shape of a model config (configs/models/<model>.json)."""
    with open(os.path.join(ROOT, "configs", "models", f"{model}.json")) as f:
        c = json.load(f)
    return dict(h=c["hidden_dim"], nq=c["num_heads"], nk=c["num_kv_heads"], hd=c["head_dim"],
                m=c["intermediate_dim"], L=c["num_layers"], V=c["vocab_size"],
                E=c.get("total_experts", 1), k=c.get("active_experts", 1))


class _Dims(dict):
    def __missing__(self, model):
        self[model] = model_dims(model)
        return self[model]


MODEL_DIMS = _Dims()  # executed FLOPs per token per decoder layer / head (fwd); see DESIGN.md
# pinned host<->device copy rates measured on this pool's B200 boxes, CUDA-event
# timed (tools/transfer_probe.py -> profiles/r02_transfer_probe.json): one
# direction alone, and both at once (total)
PCIE_H2D_GBS, PCIE_D2H_GBS, PCIE_BIDIR_GBS = 55.4, 56.4, 96.2


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return j["bf16_tflops"], j.get("bf16_tflops_sustained", j["bf16_tflops"]), j["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def ncu_gemm_traffic():
    """DRAM bytes of the captured tcgen05 GEMM launch (ncu --set full, committed
    under profiles/), with that launch's algorithmic bytes for comparison."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_full.json")), reverse=True):
        try:
            for r in json.load(open(path)):
                if "gemm_gu_fwd" in r.get("report", "") and r.get("dram_bytes"):
                    # the capture is tools/bench_gemm.py gu_fwd: 4096 x 24576 x 4096 bf16
                    algo = 2 * (4096 * 4096 + 24576 * 4096 + 4096 * 24576)
                    return {"traffic": int(r["dram_bytes"]), "algorithmic_bytes": algo,
                            "launch": "gate_up fwd 4096x24576x4096",
                            "source": os.path.relpath(path, ROOT)}
        except Exception:
            continue
    return None


def step_flops(d, seq, tokens, recompute_layers, lora_rank=0):
    """Executed FLOPs of one step: 3x fwd per layer (+1 fwd for recomputed
    layers), causal attention, head fwd+dgrad+wgrad. MoE layers: router +
    k of E experts per token. LoRA: no base wgrad (frozen), plus the rank-r
    adapter GEMMs (2 fwd + 4 bwd per adapted linear: the four linears of a
    dense layer, the attention projections of an MoE layer)."""
    qkvd = (d["nq"] + 2 * d["nk"]) * d["hd"]
    moe = d.get("E", 1) > 1
    mlp = d["k"] * 3 * d["h"] * d["m"] + d["h"] * d["E"] if moe else 3 * d["h"] * d["m"]
    lin = 2 * tokens * (d["h"] * qkvd + d["nq"] * d["hd"] * d["h"] + mlp)
    attn = 2 * d["nq"] * d["hd"] * tokens * seq  # causal fwd (QK^T + PV)
    layer_fwd = lin + attn
    head = 2 * tokens * d["h"] * d["V"]
    if lora_rank:
        io = (d["h"] + qkvd) + (d["nq"] * d["hd"] + d["h"])
        if not moe:
            io += (d["h"] + 2 * d["m"]) + (d["m"] + d["h"])
        adapters = 2 * tokens * lora_rank * io  # one pass of X A^T + U B^T over the adapted linears
        per_layer = 2 * lin + 3.5 * attn + 3 * adapters
        return d["L"] * per_layer + recompute_layers * (layer_fwd + adapters) + 2 * head
    return d["L"] * 3 * layer_fwd + recompute_layers * layer_fwd + 3 * head


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons, power = [], 0.0, set(), []
        for line in self.f:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9 or not parts[0].isdigit() or int(parts[0]) >= self.gpus:
                continue
            try:
                clk, cmax, pw = float(parts[1]), float(parts[2]), float(parts[3])
            except ValueError:
                continue
            mx = max(mx, cmax)
            power.append(pw)
            if pw > 300:  # under load
                sm.append(clk)
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"], parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(power),
                "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------------------- CPU side
def cpu_step_sample(model="qwen3-8b", tokens=32, steps=2, warmup=1, threads=None,
                    budget_s=None):
    """Bounded CPU sample of the training step, timed end to end (no
    assembly from parts): the fp32 CPU oracle's math (oracle/step_oracle.py:
    Qwen3 decoder layers, RMSNorm, RoPE, GQA attention, SwiGLU, LM head + CE)
    on all host cores, for a model of the named architecture at FULL depth —
    embedding, L decoder layers, LM head — whose L decoder layers share ONE
    weight set (the FLOPs per token equal the real model's; host memory is
    1/L of it). One sampled step = forward + backward of one sequence of
    `tokens` tokens (gradients accumulated in place). The optimizer is not in
    the sample: AdamW over 8.2B parameters once per 65,536-token step is
    < 0.2 % of the CPU step's time. The short sequence also makes attention
    cheaper than at seq 4096, so the CPU throughput is, if anything,
    overstated. Returns per-step seconds of the timed steps (the first
    `warmup` are not timed; `budget_s` stops the timed loop early)."""
    import torch
    from oracle import step_oracle as O
    threads = threads or os.cpu_count()
    torch.set_num_threads(threads)
    s = O.Shape.from_config(model)
    a = 0.02 * 3 ** 0.5  # uniform with std 0.02 (normal_ is single-threaded)

    def mat(*shape):
        return torch.empty(shape).uniform_(-a, a).requires_grad_(True)
    lp = {n: (torch.ones(sh).requires_grad_(True) if len(sh) == 1 else mat(*sh))
          for n, sh in O.layer_param_shapes(s)}
    emb, wn, wh = mat(s.vocab, s.hidden), torch.ones(s.hidden).requires_grad_(True), mat(s.vocab, s.hidden)
    params = list(lp.values()) + [emb, wn, wh]
    for p in params:
        p.grad = torch.zeros_like(p)
    g = torch.Generator().manual_seed(1234)
    ids = torch.randint(0, s.vocab, (1, tokens + 1), generator=g)
    tok, lab = ids[:, :-1], ids[:, 1:]
    cos, sin = O.rope_cos_sin(tokens, s.head_dim, s.rope_theta)
    times = []
    t_start = time.perf_counter()
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        x = emb[tok]
        for _ in range(s.layers):
            x = O.decoder_layer(x, lp.__getitem__, "", s, cos, sin)
        x = O.rms(x, wn, s.eps)
        loss = torch.nn.functional.cross_entropy((x @ wh.t()).view(-1, s.vocab),
                                                 lab.reshape(-1), reduction="mean")
        loss.backward()
        if i >= warmup:
            times.append(time.perf_counter() - t0)
        if budget_s and time.perf_counter() - t_start > budget_s and times:
            break
    return times, threads, s


def sample_desc(model, tokens, L):
    return (f"fp32 CPU oracle (oracle/step_oracle.py math, torch CPU): full-depth {model} "
            f"({L} decoder layers sharing one weight set, embedding, LM head) forward + "
            f"backward of one {tokens}-token sequence, timed end to end per step (optimizer "
            f"excluded: <0.2% of a 65,536-token CPU step); tokens/s = {tokens} / step time")


def reference_planner_times(model, seq, M):
    """The reference's own CPU path (oracle/_ref = the reference headers built
    from /root/reference): optimal_partition + synthesize + simulate for N =
    1, 2, 4, 8 on the model's cost table (built by this repo's bit-exact
    cost model: the reference ships no qwen3-8b config), single-threaded by
    construction; mem_limit 0.9 x 180 GB."""
    import ctypes
    from paper_2604_27085_b200.planner import Planner
    so = os.path.join(ROOT, "oracle", "_ref", "libref_planner.so")
    if not os.path.exists(so):
        return {"unavailable": "oracle/_ref not built"}
    ours = Planner()
    costs = ours.layer_costs(ours.load_model(model), seq, 1, ours.load_gpu("b200"), True)
    ref = Planner(ctypes.CDLL(so), prefix="ref_")
    out = {}
    for N in (1, 2, 4, 8):
        t0 = time.perf_counter()
        plan = ref.optimal_partition(costs, N, M, int(0.9 * 180e9))
        durs = ref.slot_durations(plan, costs)
        sched = ref.synthesize("roundpipe", N, M, 0, 7, durs)
        sim = ref.simulate(sched, False)
        wall = time.perf_counter() - t0
        bub = ref.interior_bubble(sim.timeline, N, 2, 4)[0]
        out[f"n{N}"] = {"wall_ms": round(wall * 1e3, 3), "slots": plan.num_slots(),
                        "tasks": len(sched.tasks), "sim_interior_bubble": round(bub, 5)}
    out["cores"] = 1
    out["what"] = "reference partition + synthesize (7 iterations) + simulate, 1 host core"
    return out


def c1_cpu_tokens_per_s(steps=2):
    """C1 (BASELINE configs[0]: tiny, seq 256, M=4) one full RoundPipe step end
    to end on the CPU oracle (sync), all host cores."""
    import torch
    from oracle import step_oracle as O
    torch.set_num_threads(os.cpu_count())
    s = O.Shape.from_config("tiny")
    o = O.StepOracle(s, O.init_params(s, seed=0), mode="sync", lr=1e-3)
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    o.step(tok, lab)
    t0 = time.perf_counter()
    for _ in range(steps):
        o.step(tok, lab)
    dt = (time.perf_counter() - t0) / steps
    return {"tokens_per_s": round(4 * 256 / dt, 1), "step_s": round(dt, 3),
            "cores": os.cpu_count(), "config": "tiny h256 L4 V32768, seq 256, M=4, sync"}


def run_reference(args):
    tokens = args.cpu_tokens
    # bounded so the whole --steps K --warmup W run ends within a few minutes
    times, threads, s = cpu_step_sample(args.model, tokens, steps=args.steps, warmup=args.warmup,
                                        budget_s=240)
    step_s = statistics.mean(times)
    v = tokens / step_s
    extras = {}
    try:
        extras["reference_planner"] = reference_planner_times(args.model, args.seq,
                                                              args.micro_batches)
    except Exception as e:  # report, never fail the line
        extras["reference_planner"] = {"error": str(e)[:200]}
    try:
        extras["c1_cpu_step"] = c1_cpu_tokens_per_s()
    except Exception as e:
        extras["c1_cpu_step"] = {"error": str(e)[:200]}
    sample = sample_desc(args.model, tokens, s.layers)
    line = {"impl": "reference", "metric": metric_name(args), "value": round(v, 3),
            "unit": "tokens/s", "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
            "ms_per_step": round(step_s * 1e3, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args),
            "cpu_baseline": {"value": round(v, 3), "unit": "tokens/s", "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            **extras}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU side
MODEL_NAMES = {"qwen3-8b": "Qwen3-8B", "qwen3-1.7b": "Qwen3-1.7B", "tiny": "tiny Qwen3",
               "qwen3-235b-a22b-l8": "Qwen3-235B-A22B (8 of 94 layers)",
               "qwen3-235b-a22b-l6": "Qwen3-235B-A22B (6 of 94 layers)",
               "qwen3-32b-l12": "Qwen3-32B (12 of 64 layers)"}


def baseline_config(args):
    """Which BASELINE.json config the run measures."""
    if args.model.startswith("qwen3-235b-a22b"):
        return "BASELINE configs[4] at reduced depth: MoE LoRA, weights streamed from pinned host"
    if args.model.startswith("qwen3-32b"):
        return ("BASELINE configs[3]" + ("" if args.model == "qwen3-32b" else " at reduced depth")
                + ": auto layer partitioning")
    if args.model == "qwen3-1.7b":
        return "BASELINE configs[1]"
    if args.model == "qwen3-8b" and not args.lora_rank:
        return "BASELINE configs[2]"
    return "not a BASELINE config"


def metric_name(args):
    return (f"fine-tune tokens/s ({MODEL_NAMES.get(args.model, args.model)} "
            f"seq{args.seq // 1024 if args.seq >= 1024 else args.seq}"
            f"{'K' if args.seq >= 1024 else ''}, RoundPipe)")


def weight_gb(model):
    d = MODEL_DIMS[model]
    qkvd = (d["nq"] + 2 * d["nk"]) * d["hd"]
    mlp = 3 * d["h"] * d["m"] * d.get("E", 1) + (d["h"] * d["E"] if d.get("E", 1) > 1 else 0)
    layer = d["h"] * qkvd + d["nq"] * d["hd"] * d["h"] + mlp
    return 2 * (d["L"] * layer + 2 * d["V"] * d["h"]) / 1e9


def config_dict(args, resident=None, mode=None):
    resident = args.resident_optimizer if resident is None else resident
    mode = mode or args.mode
    kind = f"LoRA r={args.lora_rank} fine-tune" if args.lora_rank else "full fine-tune"
    name = MODEL_NAMES.get(args.model, args.model)
    return {"workload": (f"{name} {kind} seq {args.seq // 1024 if args.seq >= 1024 else args.seq}"
                         f"{'K' if args.seq >= 1024 else ''} with "
                         + ("fp32 AdamW states HBM-resident for the groups that fit (rest "
                            "host-offloaded)" if resident else "host-offloaded Adam states")
                         + f" and activation recompute ({baseline_config(args)}): b=1, "
                         f"M={args.micro_batches} micro-batches/step, "
                         f"RoundPipe-{'async' if mode == 'async' else 'sync'}, N={args.gpus}"),
            "partitioner_residency_factor": args.residency_factor,
            "weights": ("published through the pinned bf16 master and re-uploaded every "
                        "iteration" if args.host_publish or args.gpus > 1 else
                        "AdamW results published into the device weights in place (one GPU)"),
            "model": args.model, "global_batch": args.micro_batches, "seq_len": args.seq,
            "tokens_per_step": args.micro_batches * args.seq,
            "optimizer_state": "hbm-resident where it fits" if resident else "pinned host (streamed)",
            "parallelism": f"roundpipe-{args.gpus}",
            "l2": f"inputs larger than L2 ({weight_gb(args.model):.1f} GB of bf16 weights "
                  "read per step)"}


def measure(args, resident, mode, steps, warmup, profile=False, report_dir=None, clocks=True):
    """One RoundPipe runtime, `warmup` untimed + `steps` timed steps."""
    import torch

    from paper_2604_27085_b200.planner import Planner
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe

    t_setup = time.time()
    rt = RoundPipe(args.model, seq_len=args.seq, micro_batch=1, micro_batches=args.micro_batches,
                   num_gpus=args.gpus, async_optimizer=mode == "async", adam=AdamW(lr=1e-5),
                   record_timeline=True, lora_rank=args.lora_rank, lora_alpha=args.lora_alpha,
                   host_publish=args.host_publish, residency_factor=args.residency_factor,
                   resident_state_gb=-1.0 if resident else 0.0)
    setup_s = time.time() - t_setup
    d = MODEL_DIMS[args.model]
    g = torch.Generator().manual_seed(1234)
    ids = torch.randint(0, d["V"], (args.micro_batches, 1, args.seq + 1), generator=g)
    tokens = ids[..., :-1].contiguous().int().numpy()
    labels = ids[..., 1:].contiguous().int().numpy()
    tokens_step = args.micro_batches * args.seq
    losses = []
    for _ in range(warmup):
        losses.append(rt.forward_backward(tokens, labels))
        rt.step()
    rt.sync()
    rt.clear_timeline()
    st0 = rt.stats()
    with ClockSampler(args.gpus if clocks else 0) as clk:
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        w0 = time.perf_counter()
        # non-blocking forward_backward: step t's loss is read (D2H) while
        # t+1 is enqueued, so S=1 plans on N>1 GPUs overlap iterations
        prev = None
        for _ in range(steps):
            cur = rt.forward_backward_async(tokens, labels)
            rt.step()
            if prev is not None:
                losses.append(rt.loss(prev))
            prev = cur
        losses.append(rt.loss(prev))
        rt.sync()
        w1 = time.perf_counter()
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    st1 = rt.stats()
    tl = rt.timeline()
    plan, durs = rt.plan()
    pl = Planner()
    N = args.gpus
    it_lo, it_hi = warmup, warmup + steps - 1
    if mode == "async":
        lo, hi = (it_lo + 1, it_hi - 1) if steps >= 3 else (it_lo, it_hi)
        bub = pl.interior_bubble(tl, N, lo, hi)[0]
    else:  # sync: idle inside one iteration's window (middle timed iteration)
        mid = tl[tl["iteration"] == (it_lo + it_hi) // 2]
        bub = pl.idle_in_window(tl, N, int(mid["start_ns"].min()), int(mid["end_ns"].max()))[0] \
            if len(mid) else None
    whole = pl.timeline_report(tl, N).bubble_ratio  # 1 - busy / (N x span), gaps included
    sched = pl.synthesize("roundpipe" if mode == "async" else "roundpipe-sync", N,
                          args.micro_batches, 0, max(3, steps), durs)
    sim = pl.simulate(sched, mode != "async")
    sim_bub = (pl.interior_bubble(sim.timeline, N, 1, max(3, steps) - 2)[0]
               if mode == "async" else sim.bubble_ratio)
    if report_dir:  # measured timeline in the reference CLI's report schema + Gantt
        from paper_2604_27085_b200.planner import report_json
        os.makedirs(report_dir, exist_ok=True)
        rep = pl.timeline_report(tl, N)
        tag = f"{args.model}_n{N}_{mode}"
        with open(os.path.join(report_dir, f"timeline_{tag}.json"), "w") as f:
            json.dump({"measured": report_json(rep, N),
                       "simulated": {k: v for k, v in report_json(sim, N).items() if k != "events"},
                       "transfers": rt.transfer_timeline().tolist()}, f)
        with open(os.path.join(report_dir, f"gantt_{tag}.svg"), "w") as f:
            f.write(pl.render_gantt(tl, N, plan))
    prof = None
    if profile:  # one profiled step (not timed): kernel-level roofline
        rt.profile(True)
        rt.forward_backward(tokens, labels)
        rt.step()
        prof = rt.profile_read()
        rt.profile(False)
    rt.sync()
    rt.close()
    return {"ms": ms, "wall_s": w1 - w0, "steps": steps, "tokens_step": tokens_step,
            "value": steps * tokens_step / (ms * 1e-3),
            "e2e": steps * tokens_step / (w1 - w0), "st0": st0, "st1": st1, "plan": plan,
            "bubble": bub, "sim_bubble": sim_bub, "whole_run_idle": whole, "losses": losses,
            "prof": prof,
            "clocks": clk.summary() if clocks else None, "setup_s": setup_s}


def run_ours(args):
    resident = args.resident_optimizer
    r = measure(args, resident, args.mode, args.steps, args.warmup, profile=True,
                report_dir=args.report_dir)
    d = MODEL_DIMS[args.model]
    st0, st1, plan, prof = r["st0"], r["st1"], r["plan"], r["prof"]
    burst, sustained, hbm, src = peaks()
    gemm = prof["gemm"]
    gemm_tf = gemm["work"] / (gemm["ms"] * 1e-3) / 1e12 if gemm["ms"] else 0.0
    attn = prof["attention"]
    attn_tf = attn["work"] / (attn["ms"] * 1e-3) / 1e12 if attn["ms"] else 0.0
    hbmk = prof["hbm_kernels"]
    adam = prof["adamw"]
    steps = args.steps
    h2d = (st1["h2d_bytes"] - st0["h2d_bytes"]) / steps
    d2h = (st1["d2h_bytes"] - st0["d2h_bytes"]) / steps
    p2p = (st1["p2p_bytes"] - st0["p2p_bytes"]) / steps
    recompute = sum(x.size() for x in plan.bwd_stages)
    flops = step_flops(d, args.seq, r["tokens_step"], recompute, args.lora_rank)
    t_comp = flops / (sustained * 1e12) / args.gpus
    t_link = max(h2d / (PCIE_H2D_GBS * 1e9), d2h / (PCIE_D2H_GBS * 1e9),
                 (h2d + d2h) / (PCIE_BIDIR_GBS * 1e9)) / args.gpus
    roof_tps = r["tokens_step"] / max(t_comp, t_link)
    traffic = ncu_gemm_traffic()
    line = {
        "metric": metric_name(args), "value": round(r["value"], 2), "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": round(r["ms"] / steps, 2), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded uniform token ids; random-init N(0,0.02) weights)",
        "config": config_dict(args),
        "clocks": r["clocks"],
        "e2e": {"value": round(r["e2e"], 2), "unit": "tokens/s",
                "h2d_bytes_per_step": int(r["tokens_step"] * 8), "d2h_bytes_per_step": 4,
                "streamed_h2d_bytes_per_step": int(h2d), "streamed_d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(st1["kernels_launched"] - st0["kernels_launched"]),
        "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMM (all linear layers of the step)",
                     "achieved": round(gemm_tf, 1), "peak": sustained, "unit": "TFLOP/s",
                     "frac": round(gemm_tf / sustained, 4),
                     "traffic": (traffic or {}).get("traffic"), "traffic_detail": traffic,
                     "peak_source": f"{src} bf16_tflops_sustained (kernel inside a long step)",
                     "launches": gemm["launches"]},
        "kernels": {"attention_tflops": round(attn_tf, 1),
                    "hbm_kernels_gbs": round(hbmk["work"] / (hbmk["ms"] * 1e-3) / 1e9, 1) if hbmk["ms"] else None,
                    "adamw_gbs": round(adam["work"] / (adam["ms"] * 1e-3) / 1e9, 1) if adam["ms"] else None,
                    "ms_per_step": {k: round(v["ms"], 2) for k, v in prof.items()}},
        "step_roofline": {"flops_per_step": flops, "t_compute_ms": round(t_comp * 1e3, 1),
                          "t_link_ms": round(t_link * 1e3, 1),
                          "tokens_per_s_bound": round(roof_tps, 1),
                          "frac": round(r["value"] / roof_tps, 4),
                          "note": "slower of executed FLOPs at sustained bf16 peak and streamed "
                                  "host-link bytes at the measured PCIe H2D / D2H / bidirectional "
                                  "GB/s (profiles/r02_transfer_probe.json)"},
        "transfers": {"p2p_bytes_per_step": int(p2p), "h2d_gbs_avg": round(h2d / (r["ms"] / steps * 1e-3) / 1e9, 2),
                      "d2h_gbs_avg": round(d2h / (r["ms"] / steps * 1e-3) / 1e9, 2)},
        "bubble": {"measured": round(r["bubble"], 5) if r["bubble"] is not None else None,
                   "simulated": round(r["sim_bubble"], 5), "slots": plan.num_slots(),
                   "whole_run_idle": round(r["whole_run_idle"], 5),
                   "kind": "interior (async)" if args.mode == "async" else "in-iteration (sync)",
                   "iterations": [args.warmup, args.warmup + steps - 1]},
        "loss": {"first": r["losses"][0], "last": r["losses"][-1]},
        "setup_s": round(r["setup_s"], 1),
        "optimizer_state": {"resident_params_hbm": int(st1["resident_params"]),
                            "streamed_params_host": int(st1["params_total"] - st1["resident_params"])},
        # the runtime's device allocations by category (all workers), GB
        "hbm_gb": {k: round(v / 1e9, 2) for k, v in zip(
            ("weights_2_versions", "grads", "pending_adamw_out", "activations",
             "scratch", "checkpoints_handoffs", "optimizer_chunk_ring",
             "resident_optimizer_state"),
            st1["device_bytes"][:8])},
    }
    if not args.no_variants:
        variants = {}
        vs, vw = min(args.steps, 6), 3
        for name, res, mode in (("hbm_resident_optimizer", not resident, args.mode),
                                ("roundpipe_sync", resident, "sync" if args.mode == "async" else "async")):
            try:
                v = measure(args, res, mode, vs, vw, clocks=False)
                variants[name] = {"value": round(v["value"], 2), "unit": "tokens/s",
                                  "ms_per_step": round(v["ms"] / vs, 2), "steps": vs,
                                  "bubble": round(v["bubble"], 5) if v["bubble"] is not None else None,
                                  "simulated_bubble": round(v["sim_bubble"], 5),
                                  "whole_run_idle": round(v["whole_run_idle"], 5),
                                  "config": config_dict(args, res, mode)["workload"]}
            except Exception as e:  # report, never fail the headline
                variants[name] = {"error": str(e)[:300]}
        line["variants"] = variants
    if not args.no_cpu_baseline:
        try:
            times, threads, s = cpu_step_sample(args.model, args.cpu_tokens, steps=1, warmup=1)
            v = args.cpu_tokens / statistics.mean(times)
            line["cpu_baseline"] = {"value": round(v, 3), "unit": "tokens/s", "cores": threads,
                                    "kind": "port",
                                    "sample": sample_desc(args.model, args.cpu_tokens, s.layers)}
        except Exception as e:  # report, never fail the GPU line
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="qwen3-8b")
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--micro-batches", type=int, default=16)
    ap.add_argument("--mode", default="async", choices=["async", "sync"])
    ap.add_argument("--resident-optimizer", action="store_true",
                    help="keep the fp32 AdamW state of the groups that fit in HBM (single "
                         "device) instead of the host-offloaded BASELINE configs[2] placement")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the labelled resident-optimizer / sync comparison runs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=32,
                    help="tokens of the bounded CPU step sample (cpu_baseline / --impl reference)")
    ap.add_argument("--lora-rank", type=int, default=0,
                    help="LoRA fine-tune (base frozen, rank-r adapters); 0 = full fine-tune")
    ap.add_argument("--lora-alpha", type=float, default=0.0)
    ap.add_argument("--residency-factor", type=float, default=2.0,
                    help="the partitioner's residency factor (reference default 2.0: two "
                         "weight versions; its backward/fused stages add same-size gradients). "
                         "LoRA runs have no base-weight gradients, so 1.0 models their "
                         "backward/fused stages exactly (2 x weights)")
    ap.add_argument("--host-publish", action="store_true",
                    help="one GPU: publish every AdamW result through the pinned bf16 master "
                         "and re-upload it (the paper's path; C5's weights streamed from pinned "
                         "host memory) instead of writing it into the device weights in place")
    ap.add_argument("--report-dir", default=None,
                    help="write the measured timeline (report JSON + SVG Gantt) here")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1:  # the CPU baseline is an N=1 figure; the variants are single-device
        args.no_cpu_baseline = True
        args.no_variants = True
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:  # single controller: rank 0 drives all N workers
            dist.barrier()
            dist.destroy_process_group()
            return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
