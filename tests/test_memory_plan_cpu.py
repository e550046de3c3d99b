"""Device-memory plan on the host (rp_memory_plan, no GPU): the
activation-aware partition limit (the reference partitioner
ignores activations, partitioner.hpp:74-80 / SPEC.md:202) and the pooled
workers' footprint (one buffer per group and worker made
Qwen3-32B at seq 8K impossible at N=8)."""
import pytest

from paper_2604_27085_b200.runtime import memory_plan

HBM = int(180e9)


def test_qwen3_32b_seq8k_fits_on_eight_b200_only_pooled():
    r = memory_plan("qwen3-32b", seq_len=8192, micro_batches=16, num_gpus=8, hbm_bytes=HBM)
    assert r["num_slots"] == 44  # the partitioner's S for C4
    assert r["total_static"] > HBM  # one buffer per group and worker: does not fit
    assert r["pooled"] == 1 and r["total_pooled"] < 0.5 * HBM
    # the partitioner planned with HBM minus what a worker holds besides parameters
    fixed = sum(r[k] for k in ("activations", "scratch", "handoff", "optimizer_ring", "workspace"))
    assert r["mem_limit_bytes"] == int(0.9 * HBM) - fixed


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_qwen3_8b_plans(N):
    r = memory_plan("qwen3-8b", seq_len=4096, micro_batches=16, num_gpus=N, hbm_bytes=HBM)
    assert r["num_slots"] == (1 if N <= 2 else 17)
    if N == 1:  # the fused stage keeps one activation set per layer (36)
        assert r["activations"] > 36 * 0.5e9
        assert r["total_static"] < HBM
    assert r["pool_peak"] <= r["static_groups"]


def test_activation_reserve_changes_the_plan_when_memory_binds():
    """A tight HBM budget: the activation-aware limit is below the parameter-only
    one, so the plan the runtime uses differs from planning on raw HBM."""
    r_aware = memory_plan("qwen3-8b", seq_len=4096, micro_batches=16, num_gpus=4, hbm_bytes=int(60e9))
    r_raw = memory_plan("qwen3-8b", seq_len=4096, micro_batches=16, num_gpus=4, hbm_bytes=int(60e9),
                        mem_limit_bytes=int(0.9 * 60e9))
    assert r_aware["mem_limit_bytes"] < r_raw["mem_limit_bytes"]
    assert r_aware["num_slots"] >= r_raw["num_slots"]


def test_qwen3_235b_moe_lora_plan():
    """BASELINE configs[4] (Qwen3-235B-A22B MoE, LoRA r=32, seq 31K) at N=8:
    the MoE layer's routed-row buffers (T*k rows) are in the activation /
    scratch accounting, adapters are the only trainable state (no device
    grads beyond them), and the partitioner's plan is the reference's S=64.
    The pooled weight peak (two iterations of a worker's slot weights: the
    LPT-windowed prefetch of t+1 under t) exceeds one B200 at this size —
    per-slot just-in-time weight windows are the recorded next step (DESIGN)."""
    r = memory_plan("qwen3-235b-a22b", seq_len=31744, micro_batches=8, num_gpus=8, hbm_bytes=HBM,
                    lora_rank=32)
    assert r["num_slots"] == 64
    assert r["pooled"] == 1 and r["pool_grads"] == 0
    T, k, m, h, E = 31744, 8, 1536, 4096, 128
    # expert-sorted MLP buffers: 3 dgu ring entries + sorted inputs/outputs + dact'
    assert r["scratch"] >= 3 * T * k * 2 * m * 2 + 2 * T * k * h * 2 + T * k * m * 2
    assert r["pool_weights"] > 180e9  # documented limit (see docstring)
