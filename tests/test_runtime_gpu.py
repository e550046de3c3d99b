"""End-to-end parity of the B200 RoundPipe step against the CPU oracle.

Config C1 (BASELINE configs[0]): tiny Qwen3-style decoder (4 layers, h256,
32K vocab), seq 256, M=4 micro-batches, weights seed 0 / std 0.02, tokens
seed 1234, AdamW lr 1e-3 betas (0.9, 0.95) wd 0. Sync and async
(staleness-1) modes, 3 steps, on
  * N=1 (the partitioner's single fused stage), and
  * N=4 logical workers with a supplied uniform cost table (S=7: fwd [0..2],
    [3], fused [4], bwd [3], [2], [1], [0]) so the dispatcher, hand-offs,
    checkpoints and recompute all run; workers share the one B200.
Tolerances (bf16 compute vs fp32 oracle):
  loss rel <= 2e-3; per-tensor grads rel-L2 <= 2e-2 and cosine >= 0.999
  (tensors with norm > 1e-6); fp32 master after 3 steps rel-L2 <= 2e-2 and
  cosine(dW_gpu, dW_oracle) >= 0.98 for the accumulated update dW of every
  weight matrix (rel-L2 only for the 64..4096-element norm vectors). (AdamW
  normalises every element's step to ~lr, so elements whose gradient sits
  below bf16 noise move by +-lr either way; at this config's lr 1e-3 on
  0.02-scale weights — 5 % of a weight per step — that alone gives ~1e-2
  rel-L2 after 3 steps independent of gradient error: measured 7.2e-3 sync,
  1.36e-2 async. tests/test_runtime_8b_gpu.py holds the 8B-width step to
  3e-3 at lr 1e-4.)
Schedule parity is exact: the measured timeline's task list equals the
reference dispatcher's (round, slot, mb, gpu) sequence per worker.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import step_oracle as O

pytestmark = pytest.mark.gpu
HP = dict(lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "step_golden.json")


def uniform_costs(L1):
    from paper_2604_27085_b200.planner import COST_DTYPE
    c = np.zeros(L1, dtype=COST_DTYPE)
    c["t_fwd_ns"], c["t_bwd_ns"], c["param_bytes"] = 1000, 3000, 1
    c["act_ckpt_bytes"] = 1
    return c


def run_case(mode, N, costs=None, steps=3, timeline=False, **rt_kw):
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    params = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=N,
                   async_optimizer=(mode == "async"),
                   adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                   costs=costs, skip_init=True, record_timeline=timeline, **rt_kw)
    rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
    losses, grads0 = [], None
    for it in range(steps):
        losses.append(rt.forward_backward(tok.numpy(), lab.numpy()))
        if it == 0:
            grads0 = rt.read_state(s.layers, which=2)
        rt.step()
    rt.sync()
    master = rt.read_state(s.layers, which=0)
    tl = rt.timeline() if timeline else None
    plan = rt.plan()
    rt.close()
    return losses, grads0, master, tl, plan


def oracle_case(mode, steps=3):
    s = O.Shape.from_config("tiny")
    o = O.StepOracle(s, O.init_params(s, seed=0), mode=mode, **HP)
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    losses, g0 = [], None
    for it in range(steps):
        losses.append(o.step(tok, lab))
        if it == 0:
            g0 = {k: v.clone() for k, v in o.last_grads.items()}
    return losses, g0, o.master_fp32()


_ORACLE = {}


def oracle(mode):
    if mode not in _ORACLE:
        _ORACLE[mode] = oracle_case(mode)
    return _ORACLE[mode]


def check(mode, losses, grads0, master):
    ol, og, om = oracle(mode)
    with open(GOLDEN) as f:
        gold = json.load(f)[mode]
    for a, b, c in zip(losses, ol, gold["losses"]):
        assert abs(b - c) / abs(c) < 1e-5  # oracle reproduces its pinned golden
        assert abs(a - b) / abs(b) < 2e-3, (losses, ol)
    gworst = ("", 0.0)
    for k, ref in og.items():
        g = torch.from_numpy(np.asarray(grads0[k])).reshape(ref.shape)
        rn = ref.norm().item()
        if rn < 1e-6:
            continue
        rel = (g - ref).norm().item() / rn
        cos = torch.nn.functional.cosine_similarity(g.flatten(), ref.flatten(), dim=0).item()
        gworst = max(gworst, (k, rel), key=lambda kv: kv[1])
        assert rel < 2e-2 and cos > 0.999, (k, rel, cos)
    print(mode, "worst grad rel-L2", gworst)
    worst, cosd = {}, {}
    init = O.init_params(O.Shape.from_config("tiny"), seed=0)
    for k, ref in om.items():
        w = torch.from_numpy(np.asarray(master[k])).reshape(ref.shape)
        worst[k] = (w - ref).norm().item() / ref.norm().item()
        d_gpu, d_ref = (w - init[k]).flatten(), (ref - init[k]).flatten()
        if d_ref.norm() > 0 and ref.dim() == 2:  # matrices; norm vectors are sign-noise
            cosd[k] = torch.nn.functional.cosine_similarity(d_gpu, d_ref, dim=0).item()
    print(mode, "losses", losses, "oracle", ol)
    print(mode, "worst master rel-L2", max(worst.items(), key=lambda kv: kv[1]),
          "worst update cosine", min(cosd.items(), key=lambda kv: kv[1]))
    assert max(worst.values()) < 2e-2, max(worst.items(), key=lambda kv: kv[1])
    assert min(cosd.values()) > 0.98, min(cosd.items(), key=lambda kv: kv[1])


_GPU_GRADS = {}


def test_pooled_workers_hold_their_working_set_only():
    """Pooled N=4 / S=7 workers allocate less device memory than one buffer
    per group and worker, give the same losses and grads as the static
    allocation (same kernels, other addresses), and recycle their slabs
    (a second run of steps allocates nothing new)."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    params = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    out = {}
    for pooled in (False, True):
        rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=4,
                       async_optimizer=True, adam=AdamW(**HP), costs=uniform_costs(5),
                       skip_init=True, pooled=pooled, resident_state_gb=0.0)
        rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
        losses = []
        # with gcd(S, N) = 1 a worker's set of slots repeats every N = 4
        # iterations: the pool reaches its steady size within the first N
        # (measured: 186, 292, 380, 449 MB, then 449 MB for 10 more iterations)
        for it in range(8):
            losses.append(rt.forward_backward(tok.numpy(), lab.numpy()))
            if it == 0:
                g = rt.read_state(s.layers, which=2)
            rt.step()
            if it == 3:
                rt.sync()
                st2 = rt.stats()
        rt.sync()
        st = rt.stats()
        rt.close()
        out[pooled] = (losses, g, st, st2)
    (l0, g0, st0, _), (l1, g1, st1, st1b) = out[False], out[True]
    for a, b in zip(l0, l1):
        assert abs(a - b) / abs(a) < 1e-5, (l0, l1)
    for k in g0:
        n = np.linalg.norm(g0[k])
        if n > 1e-6:
            assert np.linalg.norm(g1[k] - g0[k]) / n < 1e-3, k
    static = sum(st0["device_bytes"][c] for c in (0, 1, 2, 5))
    pooled_b = sum(st1["device_bytes"][c] for c in (0, 1, 2, 5))
    print("static", static, "pooled", pooled_b, "pool peak/worker", st1["pool_peak_bytes"])
    assert 0 < pooled_b < static
    assert st1["pool_bytes"] == st1b["pool_bytes"]  # steady state: slabs recycled


def test_multi_worker_grads_match_single_fused_stage():
    """The 4-worker / 7-slot execution (hand-offs, checkpoints, recompute)
    computes the same gradients as the single fused stage on the same GPU:
    only atomic-summation order differs -> rel-L2 <= 1e-2 per tensor."""
    _, g1, _, _, _ = run_case("sync", 1, steps=1)
    _, g4, _, _, _ = run_case("sync", 4, costs=uniform_costs(5), steps=1)
    worst = max(((k, float(np.linalg.norm(g4[k] - g1[k]) / max(np.linalg.norm(g1[k]), 1e-30)))
                 for k in g1 if np.linalg.norm(g1[k]) > 1e-6), key=lambda kv: kv[1])
    print("N=4 vs N=1 worst grad rel-L2", worst)
    assert worst[1] < 1e-2, worst


VARIANTS = {"hbm": {}, "streamed": {"resident_state_gb": 0.0},
            "pipelined": {"fused_pipeline": True},
            # LM head in 128-row chunks: the multi-chunk logits loop (wgrad
            # accumulation across chunks) and the unfused SwiGLU kernels
            "chunked_head": {"logits_rows": 128, "unfused_swiglu": True}}


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("mode", ["sync", "async"])
def test_step_parity_single_fused_stage(mode, variant):
    """Single fused stage; the fp32 optimizer state either resident in free HBM
    (single-device default) or streamed from pinned host memory every step;
    'pipelined' runs micro-batch k+1's forward beside k's backward;
    'chunked_head' runs the LM head + CE over two 128-row logits chunks."""
    losses, g0, master, _, (plan, durs) = run_case(mode, 1, **VARIANTS[variant])
    assert plan.num_slots() == 1 and plan.fused_stage.first == 0
    check(mode, losses, g0, master)


@pytest.mark.parametrize("pooled", [False, True])
@pytest.mark.parametrize("mode", ["sync", "async"])
def test_step_parity_four_workers_seven_slots(mode, pooled):
    """pooled: every worker allocates weights / grads / AdamW output /
    checkpoints on demand from its pool and returns them after their last
    use (the multi-GPU memory mode, RP_RT_POOLED)."""
    costs = uniform_costs(5)
    losses, g0, master, tl, (plan, durs) = run_case(mode, 4, costs=costs, timeline=True,
                                                    pooled=pooled)
    assert plan.num_slots() == 7
    assert [(r.first, r.last) for r in plan.fwd_stages] == [(0, 2), (3, 3)]
    assert (plan.fused_stage.first, plan.fused_stage.last) == (4, 4)
    check(mode, losses, g0, master)
    # schedule parity: measured tasks == reference dispatch list, per worker
    from paper_2604_27085_b200.planner import Planner
    ref = Planner().synthesize("roundpipe" if mode == "async" else "roundpipe-sync",
                               4, 4, 4, 3, durs)
    exp = [(t["iteration"], t["round"], t["slot"], t["mb"], t["gpu"]) for t in ref.tasks]
    got = [(e["iteration"], e["round"], e["slot"], e["mb"], e["gpu"]) for e in tl]
    assert got == exp
    for g in range(4):  # FIFO per worker: measured intervals do not overlap
        ev = tl[tl["gpu"] == g]
        assert np.all(ev["start_ns"][1:] >= ev["end_ns"][:-1] - 1000)


@pytest.mark.parametrize("resident", ["hbm", "streamed"])
@pytest.mark.parametrize("mode", ["async", "sync"])
def test_checkpoint_resume(mode, resident, tmp_path):
    """Host-state checkpoint: save after 2 steps, continue 2;
    a fresh runtime resumed from the file reproduces steps 3-4 (losses and the
    fp32 master), including async mode's unpublished staleness-1 update."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    params = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, 4, 1, 256)

    def make():
        rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=1,
                       async_optimizer=(mode == "async"),
                       adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                       skip_init=True, resident_state_gb=0.0 if resident == "streamed" else -1.0)
        return rt

    rt = make()
    rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
    for _ in range(2):
        rt.forward_backward(tok.numpy(), lab.numpy())
        rt.step()
    ck = str(tmp_path / "state.rpck")
    rt.save(ck)
    ref = []
    for _ in range(2):
        ref.append(rt.forward_backward(tok.numpy(), lab.numpy()))
        rt.step()
    rt.sync()
    m_ref = rt.read_state(s.layers, which=0)
    rt.close()
    rt2 = make()
    rt2.load(ck)
    got = []
    for _ in range(2):
        got.append(rt2.forward_backward(tok.numpy(), lab.numpy()))
        rt2.step()
    rt2.sync()
    m_got = rt2.read_state(s.layers, which=0)
    rt2.close()
    for a, b in zip(got, ref):
        assert abs(a - b) / abs(b) < 1e-4, (got, ref)
    for k in m_ref:
        a, b = np.asarray(m_got[k], np.float64), np.asarray(m_ref[k], np.float64)
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b) + 1e-9, k


def test_measured_costs_replan():
    """Measured cost table: a profiled step yields
    per-layer kernel times; re-planning N=4 on them with the reference
    partitioner and running that plan gives the same first-step loss."""
    from paper_2604_27085_b200.planner import Planner
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    params = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=1,
                   async_optimizer=False, adam=AdamW(**{"lr": 0.0}), skip_init=True)
    rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
    rt.profile(True)
    loss1 = rt.forward_backward(tok.numpy(), lab.numpy())
    rt.sync()
    mc = rt.measured_costs()
    rt.profile(False)
    rt.close()
    assert len(mc) == s.layers + 1
    assert (mc["t_fwd_ns"] > 0).all() and (mc["t_bwd_ns"] > mc["t_fwd_ns"]).all()
    plan = Planner().optimal_partition(mc, 4, 4)
    rt4 = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=4,
                    async_optimizer=False, adam=AdamW(**{"lr": 0.0}), costs=mc, skip_init=True)
    rt4.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
    assert rt4.plan()[0] == plan
    loss4 = rt4.forward_backward(tok.numpy(), lab.numpy())
    rt4.close()
    assert abs(loss4 - loss1) / loss1 < 1e-3


@pytest.mark.parametrize("N", [1, 4])
def test_step_parity_two_sequences_per_micro_batch_and_ignored_labels(N):
    """b = 2 sequences of 128 tokens per micro-batch (causal attention and
    RoPE positions restart per sequence) with ~15 % of the labels set to -100
    (ignored, not counted in the mean), sync mode, against the fp32 oracle;
    N=4 runs the S=7 dispatch with hand-offs and recompute."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    params = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, 4, 2, 128, seed=77)
    g = torch.Generator().manual_seed(5)
    lab = torch.where(torch.rand(lab.shape, generator=g) < 0.15, torch.full_like(lab, -100), lab)
    rt = RoundPipe("tiny", seq_len=128, micro_batch=2, micro_batches=4, num_gpus=N,
                   async_optimizer=False,
                   adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                   costs=uniform_costs(5) if N == 4 else None, skip_init=True)
    rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
    o = O.StepOracle(s, params, mode="sync", **HP)
    for it in range(2):
        got = rt.forward_backward(tok.numpy(), lab.numpy())
        if it == 0:
            g0 = rt.read_state(s.layers, which=2)
        rt.step()
        ref = o.step(tok, lab)
        if it == 0:
            ref_g = o.last_grads
        assert abs(got - ref) / ref < 2e-3, (it, got, ref)
    rt.sync()
    rt.close()
    for k in ("head.lm_head", "layers.0.qkv", "layers.3.down", "embed", "layers.1.q_norm"):
        a = torch.from_numpy(np.asarray(g0[k])).reshape(ref_g[k].shape)
        rel = ((a - ref_g[k]).norm() / ref_g[k].norm()).item()
        assert rel < 3e-2, (k, rel)


@pytest.mark.parametrize("N", [1, 2])
def test_non_blocking_forward_backward_matches_blocking(N):
    """rp_forward_backward_async + rp_loss (iteration t+1 enqueued before t's
    loss is read; token/label/loss buffers by iteration parity) gives the same
    losses as the blocking call, async optimizer, N=1 and N=2 workers (S=1:
    iterations alternate workers)."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    params = O.init_params(s, seed=0)
    batches = [O.synthetic_batch(s, 4, 1, 256, seed=100 + i) for i in range(4)]

    def make():
        rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=N,
                       async_optimizer=True,
                       adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                       skip_init=True)
        rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
        return rt
    rt = make()
    ref = []
    for tok, lab in batches:
        ref.append(rt.forward_backward(tok.numpy(), lab.numpy()))
        rt.step()
    rt.close()
    rt = make()
    got, prev = [], None
    for tok, lab in batches:
        cur = rt.forward_backward_async(tok.numpy(), lab.numpy())
        rt.step()
        if prev is not None:
            got.append(rt.loss(prev))
        prev = cur
    got.append(rt.loss(prev))
    with pytest.raises(Exception):
        rt.loss(0)  # only the two most recent iterations are held
    rt.sync()
    rt.close()
    for a, b in zip(got, ref):
        assert abs(a - b) / abs(b) < 1e-4, (got, ref)


@pytest.mark.parametrize("N", [1, 4])
def test_lora_step_parity(N):
    """LoRA: rank-16 adapters on the four linears
    of every layer, alpha 32, base weights frozen and streamed; 3 sync steps vs
    the fp32 oracle with PEFT semantics (only adapters train). Loss rel <=
    2e-3, adapter grads rel-L2 <= 3e-2, adapters after 3 AdamW steps cosine of
    the update >= 0.98, base weights bit-unchanged."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    r, alpha = 16, 32.0
    params = O.init_params(s, seed=0)
    params.update(O.init_lora_params(s, r, seed=3, std_a=0.02, std_b=0.02))
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=N,
                   async_optimizer=False,
                   adam=AdamW(HP["lr"], HP["betas"], HP["eps"], HP["weight_decay"]),
                   costs=uniform_costs(5) if N == 4 else None, skip_init=True,
                   lora_rank=r, lora_alpha=alpha)
    rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
    o = O.StepOracle(s, params, mode="sync", lora_scale=alpha / r, **HP)
    for it in range(3):
        got = rt.forward_backward(tok.numpy(), lab.numpy())
        if it == 0:
            g0 = rt.read_state(s.layers, which=2)
        rt.step()
        ref = o.step(tok, lab)
        if it == 0:
            ref_g = o.last_grads
        assert abs(got - ref) / ref < 2e-3, (it, got, ref)
    rt.sync()
    w = rt.read_state(s.layers, which=1)
    m = rt.read_state(s.layers, which=0)
    rt.close()
    om = o.master_fp32()
    for l in (0, 3):
        for n in ("qkv_lora_A", "qkv_lora_B", "o_lora_B", "gate_up_lora_A", "down_lora_B"):
            k = f"layers.{l}.{n}"
            a = torch.from_numpy(np.asarray(g0[k])).reshape(ref_g[k].shape)
            rel = ((a - ref_g[k]).norm() / ref_g[k].norm()).item()
            assert rel < 3e-2, (k, rel)
            du = torch.from_numpy(np.asarray(m[k])).reshape(om[k].shape) - params[k]
            dr = om[k] - params[k]
            cos = float((du * dr).sum() / (du.norm() * dr.norm()))
            assert cos > 0.98, (k, cos)
        for n in ("qkv", "down", "input_norm"):  # frozen base
            k = f"layers.{l}.{n}"
            assert np.array_equal(np.asarray(w[k]).reshape(-1),
                                  params[k].numpy().reshape(-1)), k
    assert np.array_equal(np.asarray(w["head.lm_head"]).reshape(-1),
                          params["head.lm_head"].numpy().reshape(-1))


def test_sync_direct_group_reads_after_repeated_forward(tmp_path):
    """Sync mode, single device, HBM-resident groups publishing in place:
    forward_backward twice without step() in between, then read weights,
    grads and a checkpoint (the bf16 readback wanted version ==
    iter and threw). The bf16 weights read back are bf16(fp32 master)."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    params = O.init_params(s, seed=0)
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=1,
                   async_optimizer=False, adam=AdamW(**HP), skip_init=True)
    rt.load_state({k: v.numpy() for k, v in params.items()}, s.layers)
    assert rt.stats()["resident_params"] > 0
    rt.forward_backward(tok.numpy(), lab.numpy())
    rt.step()
    rt.forward_backward(tok.numpy(), lab.numpy())
    rt.forward_backward(tok.numpy(), lab.numpy())  # no step() in between
    g = rt.read_state(s.layers, which=2)
    w16 = rt.read_state(s.layers, which=1)
    m32 = rt.read_state(s.layers, which=0)
    rt.save(str(tmp_path / "ck.rpck"))
    rt.close()
    assert np.isfinite(g["layers.0.qkv"]).all() and np.abs(g["layers.0.qkv"]).sum() > 0
    for k in ("layers.0.qkv", "head.lm_head", "embed"):
        ref = torch.from_numpy(np.asarray(m32[k])).to(torch.bfloat16).float().numpy()
        assert np.array_equal(np.asarray(w16[k]), ref), k


def test_out_of_range_ids_are_rejected():
    """Token ids outside [0, V) and labels >= V are rejected before anything
    is enqueued (they reached the gather / scatter-add kernels);
    the runtime stays usable afterwards."""
    from paper_2604_27085_b200._native import NativeError
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=1,
                   async_optimizer=False, adam=AdamW(**HP))
    bad = tok.numpy().copy()
    bad[1, 0, 7] = s.vocab
    with pytest.raises(NativeError):
        rt.forward_backward(bad, lab.numpy())
    bad = tok.numpy().copy()
    bad[0, 0, 0] = -1
    with pytest.raises(NativeError):
        rt.forward_backward(bad, lab.numpy())
    badl = lab.numpy().copy()
    badl[3, 0, 255] = s.vocab + 5
    with pytest.raises(NativeError):
        rt.forward_backward(tok.numpy(), badl)
    with pytest.raises(ValueError):
        rt.forward_backward(tok.numpy(), lab.numpy()[:2])
    loss = rt.forward_backward(tok.numpy(), lab.numpy())
    rt.close()
    assert np.isfinite(loss) and abs(loss - np.log(s.vocab)) < 0.5


@pytest.mark.parametrize("N", [1, 4])
def test_destroy_releases_device_memory(N):
    """rp_runtime_destroy frees every device allocation of every worker
    (only the resident state was freed), so creating and
    destroying runtimes in one process does not leak HBM."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    torch.cuda.synchronize()

    def cycle():
        rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=N,
                       async_optimizer=True, adam=AdamW(**HP),
                       costs=uniform_costs(5) if N == 4 else None)
        rt.forward_backward(tok.numpy(), lab.numpy())
        rt.step()
        rt.sync()
        rt.close()
    cycle()  # first cycle: kernel workspaces, module loading
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(3):
        cycle()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < (64 << 20), (free0, free1)


@pytest.mark.parametrize("N", [1, 4])
def test_memory_plan_matches_the_runtime_allocation(N):
    """rp_memory_plan (host-only byte formulas) against the runtime's own
    allocation accounting for the same configuration."""
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe, memory_plan
    kw = dict(seq_len=256, micro_batch=1, micro_batches=4, num_gpus=N, async_optimizer=True)
    rt = RoundPipe("tiny", adam=AdamW(**HP), costs=uniform_costs(5) if N == 4 else None,
                   resident_state_gb=0.0, **kw)
    st = rt.stats()
    S = rt.plan()[0].num_slots()
    rt.close()
    mp = memory_plan("tiny", hbm_bytes=torch.cuda.get_device_properties(0).total_memory, **kw)
    if N == 1:  # (the N=4 case ran on a supplied cost table; the plan uses the cost model)
        assert mp["num_slots"] == S
        assert st["device_bytes"][3] == mp["activations"] * N
    assert st["device_bytes"][6] == mp["optimizer_ring"] * N
    assert abs(st["device_bytes"][4] - mp["scratch"] * N) <= 0.05 * st["device_bytes"][4]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 visible B200s")
@pytest.mark.parametrize("pooled", [False, True])
def test_physical_devices_seven_slots(pooled):
    """N=4 workers on min(4, visible) physical B200s: hand-offs and
    checkpoint pushes cross devices over NVLink (cudaMemcpyPeerAsync), ready
    events are recorded on the producer's device; parity vs the oracle as
    the logical-worker case, and p2p bytes were moved."""
    losses, g0, master, tl, (plan, durs) = run_case("async", 4, costs=uniform_costs(5),
                                                    pooled=pooled)
    check("async", losses, g0, master)
    from paper_2604_27085_b200.runtime import AdamW, RoundPipe
    s = O.Shape.from_config("tiny")
    tok, lab = O.synthetic_batch(s, 4, 1, 256)
    rt = RoundPipe("tiny", seq_len=256, micro_batch=1, micro_batches=4, num_gpus=4,
                   async_optimizer=True, adam=AdamW(**HP), costs=uniform_costs(5), pooled=pooled)
    rt.forward_backward(tok.numpy(), lab.numpy())
    rt.step()
    rt.sync()
    st = rt.stats()
    rt.close()
    assert st["p2p_bytes"] > 0
