"""Benchmark: RoundPipe fine-tune step throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE configs[2], the metric's config): Qwen3-8B full fine-tune,
seq 4096, b=1, M=16 micro-batches per step (65,536 tokens), RoundPipe async
(staleness-1 optimizer), fp32 AdamW states host-offloaded in pinned memory
and streamed through the GPU, bf16 weights streamed from the pinned bf16
master every slot. Synthetic seeded token ids, random-init weights.

One JSON line (rank 0). `value` = tokens/s over exactly K steps bracketed by
full device synchronisation + CUDA events (max over ranks: the runtime is a
single controller, rank 0 drives all N workers); `e2e` = the same K steps
through the public API measured by the host clock (token/label host buffers
in, loss read back every step). `roofline` = the dominant kernel (tcgen05
GEMM) inside a profiled step vs the measured sustained bf16 peak; `bubble` =
the reference's interior_bubble on the MEASURED per-task timeline;
`cpu_baseline` = the fp32 CPU oracle (port) on a bounded sample.
--impl reference times the CPU implementation of the step (the oracle port:
the reference has no data-plane code) on all host cores.
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

MODEL_DIMS = {  # executed FLOPs per token per decoder layer / head (fwd); see DESIGN.md
    "qwen3-8b": dict(h=4096, nq=32, nk=8, hd=128, m=12288, L=36, V=151936),
    "qwen3-1.7b": dict(h=2048, nq=16, nk=8, hd=128, m=6144, L=28, V=151936),
    "tiny": dict(h=256, nq=4, nk=2, hd=64, m=768, L=4, V=32768),
}
PCIE_H2D_GBS, PCIE_D2H_GBS = 55.6, 52.9  # measured pinned copies on this pool (tools/probe_box.sh)


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
    layers), causal attention, head fwd+dgrad+wgrad. LoRA: no base wgrad
    (frozen), plus the rank-r adapter GEMMs (2 fwd + 4 bwd per linear)."""
    qkvd = (d["nq"] + 2 * d["nk"]) * d["hd"]
    lin = 2 * tokens * (d["h"] * qkvd + d["nq"] * d["hd"] * d["h"] + 3 * d["h"] * d["m"])
    attn = 2 * d["nq"] * d["hd"] * tokens * seq  # causal fwd (QK^T + PV)
    layer_fwd = lin + attn
    head = 2 * tokens * d["h"] * d["V"]
    if lora_rank:
        io = (d["h"] + qkvd) + (d["nq"] * d["hd"] + d["h"]) + (d["h"] + 2 * d["m"]) + (d["m"] + d["h"])
        adapters = 2 * tokens * lora_rank * io  # one pass of X A^T + U B^T over the 4 linears
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


def cpu_sample(model="qwen3-8b", seq=4096, M=16, threads=None, head_tokens=512):
    """Bounded sample of the step on the CPU oracle (fp32 torch, all host
    cores): one full-width decoder layer fwd+bwd at seq, the LM head + CE
    fwd+bwd on head_tokens tokens, AdamW over one layer's parameters. The
    full step time is assembled from these measured parts (L layers x M
    micro-batches, head scaled to M*seq tokens, AdamW x (L + 2 groups))."""
    import torch
    from oracle import step_oracle as O
    threads = threads or os.cpu_count()
    torch.set_num_threads(threads)
    s = O.Shape.from_config(model)
    g = torch.Generator().manual_seed(0)
    p = {}
    for n, sh in O.layer_param_shapes(s):
        p["l." + n] = (torch.ones(sh) if len(sh) == 1 else torch.randn(sh, generator=g) * 0.02)
    p = {k: v.requires_grad_(True) for k, v in p.items()}
    cos, sin = O.rope_cos_sin(seq, s.head_dim, s.rope_theta)
    x = torch.randn(1, seq, s.hidden, generator=g)
    t0 = time.perf_counter()
    y = O.decoder_layer(x, lambda n: p[n], "l.", s, cos, sin)
    y.float().pow(2).mean().backward()
    t_layer = time.perf_counter() - t0
    wh = (torch.randn(s.vocab, s.hidden, generator=g) * 0.02).requires_grad_(True)
    xh = torch.randn(head_tokens, s.hidden, generator=g)
    lab = torch.randint(0, s.vocab, (head_tokens,), generator=g)
    t0 = time.perf_counter()
    torch.nn.functional.cross_entropy(xh @ wh.t(), lab).backward()
    t_head = (time.perf_counter() - t0) * (seq / head_tokens)
    params = list(p.values())
    opt = torch.optim.AdamW(params, lr=1e-4)
    t0 = time.perf_counter()
    opt.step()
    t_adam_layer = time.perf_counter() - t0
    n_layer = sum(v.numel() for v in params)
    n_total = n_layer * s.layers + 2 * s.vocab * s.hidden
    step_s = M * (s.layers * t_layer + t_head) + t_adam_layer * n_total / n_layer
    return {"tokens_per_s": M * seq / step_s, "step_s": step_s, "threads": threads,
            "t_layer_s": t_layer, "t_head_s": t_head, "t_adam_layer_s": t_adam_layer,
            "sample_wall_s": None}


def run_reference(args):
    t0 = time.time()
    r = cpu_sample(args.model, args.seq, args.micro_batches)
    wall = time.time() - t0
    steps = []
    for _ in range(args.steps):  # every step is one bounded sample
        t1 = time.time()
        rr = cpu_sample(args.model, args.seq, args.micro_batches)
        steps.append(rr["step_s"])
        if time.time() - t1 > 120:
            break
    step_s = statistics.mean(steps) if steps else r["step_s"]
    v = args.micro_batches * args.seq / step_s
    sample = (f"fp32 CPU oracle (oracle/step_oracle.py): 1 full-width {args.model} decoder layer "
              f"fwd+bwd at seq {args.seq}, LM head+CE on 512 tokens, AdamW on one layer; step time "
              f"assembled for {args.micro_batches} micro-batches x all layers (first sample {wall:.1f}s)")
    line = {"impl": "reference", "metric": metric_name(args), "value": round(v, 3), "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": len(steps), "warmup": args.warmup,
            "ms_per_step": round(step_s * 1e3, 1), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args),
            "cpu_baseline": {"value": round(v, 3), "unit": "tokens/s", "cores": r["threads"],
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(v, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "fine-tune tokens/s (Qwen3-8B seq4K, RoundPipe)"
MODEL_NAMES = {"qwen3-8b": "Qwen3-8B", "qwen3-1.7b": "Qwen3-1.7B", "tiny": "tiny Qwen3"}


def metric_name(args):
    return (f"fine-tune tokens/s ({MODEL_NAMES.get(args.model, args.model)} "
            f"seq{args.seq // 1024 if args.seq >= 1024 else args.seq}"
            f"{'K' if args.seq >= 1024 else ''}, RoundPipe)")


def weight_gb(model):
    d = MODEL_DIMS[model]
    qkvd = (d["nq"] + 2 * d["nk"]) * d["hd"]
    layer = d["h"] * qkvd + d["nq"] * d["hd"] * d["h"] + 3 * d["h"] * d["m"]
    return 2 * (d["L"] * layer + 2 * d["V"] * d["h"]) / 1e9


def config_dict(args):
    kind = f"LoRA r={args.lora_rank} fine-tune" if getattr(args, "lora_rank", 0) else "full fine-tune"
    return {"workload": f"{args.model} {kind}, seq {args.seq}, b=1, M={args.micro_batches} "
                        f"micro-batches/step, RoundPipe-{'async' if args.mode == 'async' else 'sync'}, "
                        + ("fp32 AdamW master weights + states in pinned host memory (all streamed)"
                           if getattr(args, "host_optimizer", False) or args.gpus > 1 else
                           "fp32 AdamW master weights + states HBM-resident for the groups that "
                           "fit, the rest in pinned host memory (see optimizer_state)"),
            "model": args.model, "global_batch": args.micro_batches, "seq_len": args.seq,
            "tokens_per_step": args.micro_batches * args.seq,
            "parallelism": f"roundpipe-{args.gpus}",
            "l2": f"inputs larger than L2 ({weight_gb(args.model):.1f} GB of bf16 weights "
                  "read per step)"}


def run_ours(args):
    import numpy as np
    import torch

    from paper_2604_27085_b200.planner import Planner
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe

    t_setup = time.time()
    rt = RoundPipe(args.model, seq_len=args.seq, micro_batch=1, micro_batches=args.micro_batches,
                   num_gpus=args.gpus, async_optimizer=args.mode == "async", adam=AdamW(lr=1e-5),
                   record_timeline=True, lora_rank=args.lora_rank, lora_alpha=args.lora_alpha,
                   resident_state_gb=0.0 if args.host_optimizer else -1.0)
    setup_s = time.time() - t_setup
    d = MODEL_DIMS[args.model]
    g = torch.Generator().manual_seed(1234)
    ids = torch.randint(0, d["V"], (args.micro_batches, 1, args.seq + 1), generator=g)
    tokens = ids[..., :-1].contiguous().int().numpy()
    labels = ids[..., 1:].contiguous().int().numpy()
    tokens_step = args.micro_batches * args.seq
    losses = []
    for _ in range(args.warmup):
        losses.append(rt.forward_backward(tokens, labels))
        rt.step()
    rt.sync()
    rt.clear_timeline()
    st0 = rt.stats()
    with ClockSampler(args.gpus) as clk:
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        w0 = time.perf_counter()
        # non-blocking forward_backward: step t's loss is read (D2H) while
        # t+1 is enqueued, so S=1 plans on N>1 GPUs overlap iterations
        prev = None
        for _ in range(args.steps):
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
    # bubble on the measured timeline (reference formulas)
    pl = Planner()
    it_lo, it_hi = args.warmup, args.warmup + args.steps - 1
    if args.steps >= 3:
        bub = pl.interior_bubble(tl, args.gpus, it_lo + 1, it_hi - 1)[0]
    else:
        bub = pl.interior_bubble(tl, args.gpus, it_lo, it_hi)[0]
    sched = pl.synthesize("roundpipe" if args.mode == "async" else "roundpipe-sync", args.gpus,
                          args.micro_batches, 0, max(3, args.steps), durs)
    sim = pl.simulate(sched, args.mode != "async")
    sim_bub = (pl.interior_bubble(sim.timeline, args.gpus, 1, max(3, args.steps) - 2)[0]
               if args.mode == "async" else sim.bubble_ratio)
    if args.report_dir:  # measured timeline in the reference CLI's report schema + Gantt
        from paper_2604_27085_b200.planner import report_json
        os.makedirs(args.report_dir, exist_ok=True)
        rep = pl.timeline_report(tl, args.gpus)
        tag = f"{args.model}_n{args.gpus}_{args.mode}"
        with open(os.path.join(args.report_dir, f"timeline_{tag}.json"), "w") as f:
            json.dump({"measured": report_json(rep, args.gpus),
                       "simulated": {k: v for k, v in report_json(sim, args.gpus).items()
                                     if k != "events"},
                       "transfers": rt.transfer_timeline().tolist()}, f)
        with open(os.path.join(args.report_dir, f"gantt_{tag}.svg"), "w") as f:
            f.write(pl.render_gantt(tl, args.gpus, plan))
    # one profiled step (not timed): kernel-level roofline
    rt.profile(True)
    rt.forward_backward(tokens, labels)
    rt.step()
    prof = rt.profile_read()
    rt.profile(False)
    rt.sync()
    rt.close()

    burst, sustained, hbm, src = peaks()
    gemm = prof["gemm"]
    gemm_tf = gemm["work"] / (gemm["ms"] * 1e-3) / 1e12 if gemm["ms"] else 0.0
    attn = prof["attention"]
    attn_tf = attn["work"] / (attn["ms"] * 1e-3) / 1e12 if attn["ms"] else 0.0
    hbmk = prof["hbm_kernels"]
    adam = prof["adamw"]
    h2d = (st1["h2d_bytes"] - st0["h2d_bytes"]) / args.steps
    d2h = (st1["d2h_bytes"] - st0["d2h_bytes"]) / args.steps
    recompute = sum(r.size() for r in plan.bwd_stages)
    flops = step_flops(d, args.seq, tokens_step, recompute, args.lora_rank)
    t_comp = flops / (sustained * 1e12) / args.gpus
    t_link = max(h2d / (PCIE_H2D_GBS * 1e9), d2h / (PCIE_D2H_GBS * 1e9)) / args.gpus
    value = args.steps * tokens_step / (ms * 1e-3)
    e2e = args.steps * tokens_step / (w1 - w0)
    roof_tps = tokens_step / max(t_comp, t_link)
    gpu_launches = (st1["kernels_launched"] - st0["kernels_launched"])
    line = {
        "metric": metric_name(args), "value": round(value, 2), "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 2),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded uniform token ids; random-init N(0,0.02) weights)",
        "config": config_dict(args),
        "clocks": clk.summary(),
        "e2e": {"value": round(e2e, 2), "unit": "tokens/s",
                "h2d_bytes_per_step": int(args.micro_batches * args.seq * 8),
                "d2h_bytes_per_step": 4,
                "streamed_h2d_bytes_per_step": int(h2d), "streamed_d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(gpu_launches),
        "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMM (all linear layers of the step)",
                     "achieved": round(gemm_tf, 1), "peak": sustained, "unit": "TFLOP/s",
                     "frac": round(gemm_tf / sustained, 4),
                     "traffic": (ncu_gemm_traffic() or {}).get("traffic"),
                     "traffic_detail": ncu_gemm_traffic(),
                     "peak_source": f"{src} bf16_tflops_sustained (kernel inside a long step)",
                     "launches": gemm["launches"]},
        "kernels": {"attention_tflops": round(attn_tf, 1),
                    "hbm_kernels_gbs": round(hbmk["work"] / (hbmk["ms"] * 1e-3) / 1e9, 1) if hbmk["ms"] else None,
                    "adamw_gbs": round(adam["work"] / (adam["ms"] * 1e-3) / 1e9, 1) if adam["ms"] else None,
                    "ms_per_step": {k: round(v["ms"], 2) for k, v in prof.items()}},
        "step_roofline": {"flops_per_step": flops, "t_compute_ms": round(t_comp * 1e3, 1),
                          "t_link_ms": round(t_link * 1e3, 1),
                          "tokens_per_s_bound": round(roof_tps, 1),
                          "frac": round(value / roof_tps, 4),
                          "note": "slower of executed FLOPs at sustained bf16 peak and streamed "
                                  "host-link bytes at measured PCIe H2D/D2H GB/s"},
        "bubble": {"measured_interior": round(bub, 5), "simulated": round(sim_bub, 5),
                   "slots": plan.num_slots(), "iterations": [it_lo, it_hi]},
        "loss": {"first": losses[0], "last": losses[-1]},
        "setup_s": round(setup_s, 1),
        "optimizer_state": {"resident_params_hbm": int(st1["resident_params"]),
                            "streamed_params_host": int(st1["params_total"] - st1["resident_params"]),
                            "note": "fp32 AdamW state of the largest groups that fit in free HBM "
                                    "stays resident (single device); the rest streams from "
                                    "pinned host memory every step"},
        # the runtime's device allocations by category (all workers), GB
        "hbm_gb": {k: round(v / 1e9, 2) for k, v in zip(
            ("weights_2_versions", "grads", "pending_adamw_out", "activations",
             "scratch", "resident_optimizer_state", "optimizer_chunk_ring"),
            st1["device_bytes"][:7])},
    }
    if not args.no_cpu_baseline:
        try:
            r = cpu_sample(args.model, args.seq, args.micro_batches)
            line["cpu_baseline"] = {
                "value": round(r["tokens_per_s"], 3), "unit": "tokens/s", "cores": r["threads"],
                "kind": "port",
                "sample": (f"fp32 CPU oracle: 1 full-width {args.model} layer fwd+bwd at seq "
                           f"{args.seq}, head+CE on 512 tokens, AdamW on one layer; assembled into "
                           f"a {args.micro_batches}-micro-batch step")}
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lora-rank", type=int, default=0,
                    help="LoRA fine-tune (base frozen, rank-r adapters); 0 = full fine-tune")
    ap.add_argument("--lora-alpha", type=float, default=0.0)
    ap.add_argument("--report-dir", default=None,
                    help="write the measured timeline (report JSON + SVG Gantt) here")
    ap.add_argument("--host-optimizer", action="store_true",
                    help="keep every group's fp32 AdamW state in pinned host memory "
                         "(no HBM-resident groups): the strict host-offloaded configuration")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
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
