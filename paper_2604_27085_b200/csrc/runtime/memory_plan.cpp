// Device-memory plan of a RoundPipe runtime configuration, computed on the
// host without a GPU (rp_memory_plan), and the activation-aware memory limit
// the runtime hands the partitioner.
//
// The reference partitioner checks a stage's memory as residency x (1 fwd,
// 2 bwd) x its parameter bytes (partitioner.hpp:74-80) and
// ignores activations; the executor here subtracts what a worker holds
// besides parameters — activation sets, backward scratch, hand-off buffers,
// the optimizer chunk ring, kernel workspaces — from the HBM it gives the
// partitioner. The byte formulas mirror Runtime::alloc_worker
// (runtime.cpp) buffer by buffer; tests/test_runtime_gpu.py compares them
// with the runtime's own allocation accounting.
//
// Pooled workers (RP_RT_POOLED, N > 1) hold weights / grads / AdamW output /
// checkpoints only for their lifetime; their peak is found by replaying the
// controller's enqueue order over the dispatch list: weights of iteration t+1
// are reserved at the start of iteration t (LPT windows) and returned at the
// worker's last use in t+1, grads live from the first write until step(t),
// the AdamW output until p_copy at the start of t+1 (async), a checkpoint
// from its forward push until the recomputing slot read it.
#include <algorithm>
#include <cstring>
#include <map>
#include <tuple>

#include "runtime/runtime_internal.h"

namespace rp {
namespace rt {

WorkerBytes worker_fixed_bytes(const Shape& s, int T, int seq, int M, int MR, int S, int parities,
                               int nsets, int logits_rows, int lora_r, int64_t chunk_elems) {
  WorkerBytes b;
  const int64_t Th = (int64_t)T * s.h;
  const int64_t Tk = (int64_t)T * (s.moe() ? s.ek : 1);  // rows of the MLP buffers
  const int n_lora = s.moe() ? 2 : 4;                      // adapted linears
  const int64_t moe_set =
      s.moe() ? (int64_t)T * s.E * 4 + (int64_t)T * s.ek * 4 * 3 + Tk * 4 + (int64_t)(s.E + 1) * 4 : 0;
  const int64_t act_set = Th * 2 * 4 + (int64_t)T * s.qkvd() * 2 + (int64_t)T * s.qd() * 2 * 2 +
                          (int64_t)T * s.kd() * 2 + Tk * 2 * s.m * 2 + Tk * s.m * 2 +
                          (int64_t)T * 4 * 2 + (int64_t)T * s.nq * 4 * 2 + (int64_t)T * s.nk * 4 +
                          (lora_r ? (int64_t)n_lora * T * lora_r * 2 : 0) + moe_set;
  b.activations = act_set * nsets;
  const int64_t moe_scratch =
      s.moe() ? Tk * s.h * 2 * 2 + Tk * s.m * 2 + (int64_t)T * s.E * 2 + (int64_t)s.E * 4 * 2 +
                    Tk * 4 + Th * 4
              : 0;
  b.scratch = Th * 4 * 2 + Th * 2 * 2 + (int64_t)T * s.qkvd() * 2 * 2 +
              3LL * Tk * 2 * s.m * 2 + Th * 2 + (int64_t)T * s.m * 2 + (int64_t)T * s.qd() * 2 * 2 +
              (int64_t)T * s.kd() * 2 + (int64_t)T * s.qd() * 4 + (int64_t)T * s.nq * 4 +
              Th * 2 * 3 + (int64_t)T * 4 + (int64_t)std::min(T, logits_rows) * s.V * 2 +
              2LL * 2 * M * T * 4 + (int64_t)seq * s.hd * 4 + (lora_r ? (int64_t)T * lora_r * 2 : 0) +
              moe_scratch;
  b.handoff = S > 1 ? (int64_t)parities * MR * (Th * 2 + Th * 4) : 0;
  b.optimizer_ring = (int64_t)Gpu::kOptSlots * 3 * chunk_elems * 4;
  // per-stream kernel scratch: the fused attention backward's fp32 dQ^T
  // accumulator and split-K partials on the compute / weight-gradient streams
  b.workspace = (int64_t)T * s.qd() * 4 + 2LL * (37 * 2 * 128 * 256 * 4 + 37 * 8 * 4);
  return b;
}

int64_t WorkerBytes::fixed() const {
  return activations + scratch + handoff + optimizer_ring + workspace;
}

// Replays the controller's buffer lifetimes for `iters` iterations; returns
// the per-category peaks of the worker with the largest pooled peak.
PoolPeak pooled_peak(const Shape& s, const LayerLayout& LL, const HeadLayout& HL,
                     const roundpipe::StagePlan& plan,
                     const std::vector<roundpipe::StageSlot>& slots,
                     const roundpipe::Schedule& sched, int N, int MR, int T, bool async,
                     int lora_r, int iters) {
  const int L = s.L, ng = L + 2;
  auto n_of = [&](int g) -> int64_t {
    return g == 0 ? (int64_t)s.V * s.h : g == L + 1 ? HL.total : LL.total;
  };
  auto tn_of = [&](int g) -> int64_t {
    if (!lora_r) return n_of(g);
    return g >= 1 && g <= L ? LL.total - LL.lora_off : 0;
  };
  auto groups = [&](const roundpipe::StageSlot& ss) {
    std::vector<int> gs;
    if (ss.kind != roundpipe::StageKind::Backward && ss.layers.first == 0) gs.push_back(0);
    for (int l = ss.layers.first; l <= ss.layers.last; ++l) gs.push_back(l + 1);
    return gs;
  };
  const int64_t ck = (int64_t)T * s.h * 2;
  std::vector<int> bwd_slot_of(L, -1);
  for (const auto& sl : slots)
    if (sl.kind == roundpipe::StageKind::Backward)
      for (int l = sl.layers.first; l <= sl.layers.last; ++l) bwd_slot_of[l] = sl.index;
  const int S = (int)slots.size();
  std::vector<std::array<int64_t, 4>> cur(N, {0, 0, 0, 0}), peak_of(N, {0, 0, 0, 0});
  std::vector<int64_t> tot(N, 0), peak(N, 0);
  auto add = [&](int w, int cat, int64_t bytes) {
    cur[w][cat] += bytes;
    tot[w] += bytes;
    if (tot[w] > peak[w]) {
      peak[w] = tot[w];
      peak_of[w] = cur[w];
    }
  };
  // (w, g, version) weights held; grads (w, g, t); pend (w, g)
  std::map<std::tuple<int, int, int>, bool> wheld;
  std::map<std::pair<int, int>, int> grad_owner, pend_owner;
  auto tasks_of = [&](int t) {
    std::vector<const roundpipe::Task*> v;
    for (std::size_t i = 0; i < sched.tasks.size(); i += MR)
      if (sched.tasks[i].iteration == t) v.push_back(&sched.tasks[i]);
    return v;
  };
  auto reserve = [&](int t) {
    for (const auto* tk : tasks_of(t))
      for (int g : groups(slots[tk->slot]))
        if (!wheld.count({tk->gpu, g, t})) {
          wheld[{tk->gpu, g, t}] = true;
          add(tk->gpu, 0, n_of(g) * 2);
        }
  };
  for (int t = 0; t < iters; ++t) {
    if (async) {
      for (auto& [wg, w] : pend_owner) add(w, 2, -tn_of(wg.second) * 2);  // p_copy
      pend_owner.clear();
      reserve(t + 1);  // LPT-windowed uploads of the next iteration
    }
    const auto tv = tasks_of(t);
    std::map<std::pair<int, int>, std::size_t> last;
    for (std::size_t k = 0; k < tv.size(); ++k)
      for (int g : groups(slots[tv[k]->slot])) last[{tv[k]->gpu, g}] = k;
    for (std::size_t k = 0; k < tv.size(); ++k) {
      const auto* tk = tv[k];
      const int w = tk->gpu;
      const auto& ss = slots[tk->slot];
      for (int g : groups(ss))
        if (!wheld.count({w, g, t})) {
          wheld[{w, g, t}] = true;
          add(w, 0, n_of(g) * 2);
        }
      if (ss.kind != roundpipe::StageKind::Forward) {  // grads of the slot's groups
        std::vector<int> gg;
        for (int l = ss.layers.first; l <= std::min(ss.layers.last, L - 1); ++l) gg.push_back(l + 1);
        if (ss.layers.last == L) gg.push_back(L + 1);
        if (ss.layers.first == 0) gg.push_back(0);
        for (int g : gg)
          if (tn_of(g) > 0 && !grad_owner.count({g, t})) {
            grad_owner[{g, t}] = w;
            add(w, 1, tn_of(g) * 4);
          }
      }
      if (ss.kind == roundpipe::StageKind::Forward)  // checkpoints pushed to the recomputing worker
        for (int l = ss.layers.first; l <= ss.layers.last; ++l) {
          const int o = (int)(((int64_t)tk->round * S + bwd_slot_of[l]) % N);
          add(o, 3, ck * MR);
        }
      if (ss.kind == roundpipe::StageKind::Backward)  // checkpoints read
        for (int l = ss.layers.first; l <= ss.layers.last; ++l) add(w, 3, -ck * MR);
      for (int g : groups(ss))
        if (last[{w, g}] == k) {
          wheld.erase({w, g, t});
          add(w, 0, -n_of(g) * 2);
        }
    }
    // step(t): AdamW per group on the grad owner: output slab, grads returned
    for (auto it = grad_owner.begin(); it != grad_owner.end();) {
      if (it->first.second != t) {
        ++it;
        continue;
      }
      const int g = it->first.first, w = it->second;
      add(w, 2, tn_of(g) * 2);  // AdamW output: the trainable region
      add(w, 1, -tn_of(g) * 4);
      if (async)
        pend_owner[{w, g}] = w;
      else
        add(w, 2, -tn_of(g) * 2);  // sync: p_copy at once
      it = grad_owner.erase(it);
    }
    if (!async) reserve(t + 1);  // sync prefetch after the step
  }
  int wmax = 0;
  for (int w = 1; w < N; ++w)
    if (peak[w] > peak[wmax]) wmax = w;
  PoolPeak r;
  r.worker = wmax;
  r.total = peak[wmax];
  r.weights = peak_of[wmax][0];
  r.grads = peak_of[wmax][1];
  r.pend = peak_of[wmax][2];
  r.checkpoints = peak_of[wmax][3];
  (void)ng;
  return r;
}

Shape load_shape(const std::string& model) {
  const auto shape = roundpipe::config_io::load_shape(model);
  Shape s;
  s.h = (int)shape.cfg.hidden_dim;
  s.nq = shape.cfg.num_heads;
  s.nk = shape.cfg.num_kv_heads;
  s.hd = shape.head_dim;
  s.m = (int)shape.cfg.intermediate_dim;
  s.L = shape.cfg.num_layers;
  s.V = shape.vocab_size;
  s.theta = shape.rope_theta;
  s.eps = shape.rms_norm_eps;
  s.E = shape.cfg.total_experts;
  s.ek = shape.cfg.active_experts;
  s.norm_topk = shape.norm_topk_prob;
  if (s.moe() && (s.E > 256 || s.ek > 32 || s.ek > s.E))
    throw RtError(RP_E_INPUT, "MoE: up to 256 experts and 32 routed per token");
  return s;
}

PlanChoice choose_plan(const rp_runtime_config_t& cfg, const Shape& s, const std::string& model,
                       int64_t hbm_bytes, int logits_rows, int64_t chunk_elems) {
  PlanChoice c;
  if (cfg.costs && cfg.n_costs > 0) {
    if (cfg.n_costs != s.L + 1) throw RtError(RP_E_INPUT, "cost table must have L+1 rows");
    for (int i = 0; i < cfg.n_costs; ++i) {
      roundpipe::LayerCost lc;
      lc.t_fwd_ns = cfg.costs[i].t_fwd_ns;
      lc.t_bwd_ns = cfg.costs[i].t_bwd_ns;
      lc.param_bytes = cfg.costs[i].param_bytes;
      lc.act_ckpt_bytes = cfg.costs[i].act_ckpt_bytes;
      lc.act_full_bytes = cfg.costs[i].act_full_bytes;
      c.costs.push_back(lc);
    }
  } else {
    const auto mc = roundpipe::config_io::load_model(model);
    const auto gpu = roundpipe::config_io::load_gpu("b200");
    c.costs = roundpipe::cost_model::layer_costs(
        mc, roundpipe::Workload{cfg.seq_len, cfg.micro_batch}, gpu, true);
  }
  roundpipe::PartitionProblem p;
  p.costs = c.costs;
  p.num_gpus = cfg.num_gpus;
  p.micro_batches = cfg.micro_batches;
  p.residency_factor = cfg.residency_factor > 0 ? cfg.residency_factor : 2.0;
  const int T = cfg.seq_len * cfg.micro_batch;
  const int M = cfg.micro_batches;
  const int MR = cfg.round_micro_batches ? cfg.round_micro_batches : M;
  const int parities = cfg.num_gpus > 1 ? 2 : 1;
  auto fixed = [&](int nsets, int S) {
    return worker_fixed_bytes(s, T, cfg.seq_len, M, MR, S, parities, nsets, logits_rows,
                              cfg.lora_rank, chunk_elems);
  };
  if (cfg.mem_limit_bytes > 0) {
    p.mem_limit_bytes = cfg.mem_limit_bytes;
    c.plan = roundpipe::partitioner::optimal_partition(p);
  } else {
    // what a worker holds besides parameters comes off the partitioner's HBM
    // (SURVEY 8(f)1); the fused stage keeps one activation set per layer, so
    // grow the reserve until it covers the plan's fused stage
    int nsets = 1;
    for (int pass = 0; pass < 8; ++pass) {
      p.mem_limit_bytes = (int64_t)(0.9 * (double)hbm_bytes) - fixed(nsets, cfg.num_gpus > 1 ? 2 : 1).fixed();
      c.plan = roundpipe::partitioner::optimal_partition(p);
      const int ns = std::max(1, s.L - c.plan.fused_stage.first);
      if (ns <= nsets) break;
      nsets = ns;
    }
  }
  c.mem_limit = p.mem_limit_bytes;
  c.slots = roundpipe::scheduler::slot_table_from_plan(c.plan, c.costs);
  c.fixed = fixed(std::max(1, s.L - c.plan.fused_stage.first), (int)c.slots.size());
  return c;
}

}  // namespace rt
}  // namespace rp

// ======================================================================== C-ABI
#define RP_API extern "C" __attribute__((visibility("default")))

// Device-memory plan of a runtime configuration for one worker, on the host
// (no GPU needed): the activation-aware stage plan, the fixed per-worker
// buffers, one-buffer-per-group bytes, and the pooled peak of the worst
// worker over the first 6 iterations of the dispatch list.
RP_API int rp_memory_plan(const rp_runtime_config_t* cfg, int64_t hbm_bytes,
                          rp_memory_plan_t* out) {
  using namespace rp::rt;
  try {
    if (!cfg || !out || hbm_bytes <= 0) return RP_E_INPUT;
    const std::string model = cfg->model ? cfg->model : "qwen3-8b";
    const Shape s = load_shape(model);
    if (cfg->seq_len < 128 || cfg->seq_len % 128 || cfg->micro_batches < 1 || cfg->num_gpus < 1)
      return RP_E_INPUT;
    const int logits_rows = cfg->logits_rows ? cfg->logits_rows : 2048;
    const int64_t chunk = 32ll << 20;
    const PlanChoice pc = choose_plan(*cfg, s, model, hbm_bytes, logits_rows, chunk);
    const int N = cfg->num_gpus, M = cfg->micro_batches;
    const int MR = cfg->round_micro_batches ? cfg->round_micro_batches : M;
    const int T = cfg->seq_len * cfg->micro_batch;
    const LayerLayout LL = make_layer_layout(s, cfg->lora_rank);
    const HeadLayout HL = make_head_layout(s);
    roundpipe::ScheduleSpec spec;
    spec.kind = cfg->async_optimizer ? roundpipe::ScheduleKind::RoundPipe
                                     : roundpipe::ScheduleKind::RoundPipeSync;
    spec.num_gpus = N;
    spec.micro_batches = M;
    spec.round_micro_batches = MR;
    spec.iterations = 8;
    for (const auto& sl : pc.slots) spec.slot_durs.push_back(sl.dur_ns);
    const auto sched = roundpipe::scheduler::synthesize(spec);
    const PoolPeak pk = pooled_peak(s, LL, HL, pc.plan, pc.slots, sched, N, MR, T,
                                    cfg->async_optimizer != 0, cfg->lora_rank, 6);
    std::memset(out, 0, sizeof(*out));
    out->num_slots = (int32_t)pc.slots.size();
    out->mem_limit_bytes = pc.mem_limit;
    out->activations = pc.fixed.activations;
    out->scratch = pc.fixed.scratch;
    out->handoff = pc.fixed.handoff;
    out->optimizer_ring = pc.fixed.optimizer_ring;
    out->workspace = pc.fixed.workspace;
    int64_t groups = 0;
    // one worker publishes AdamW results into the device weights in place
    // (Runtime::publish_in_place): no AdamW output buffer
    const bool in_place = N == 1 && !(cfg->flags & RP_RT_HOST_PUBLISH);
    for (int g = 0; g < s.L + 2; ++g) {
      const int64_t n = g == 0 ? (int64_t)s.V * s.h : g == s.L + 1 ? HL.total : LL.total;
      const int64_t tn = cfg->lora_rank ? (g >= 1 && g <= s.L ? LL.total - LL.lora_off : 0) : n;
      groups += n * 2 * 2 + (in_place ? 0 : tn * 2) + tn * 4 * 2;  // 2 weight versions, AdamW output, 2 grads
    }
    const int lck = std::max(0, pc.plan.fused_stage.first);
    if (pc.slots.size() > 1) groups += (int64_t)(N > 1 ? 2 : 1) * lck * MR * T * s.h * 2;
    out->static_groups = groups;
    out->pool_worker = pk.worker;
    out->pool_peak = pk.total;
    out->pool_weights = pk.weights;
    out->pool_grads = pk.grads;
    out->pool_pend = pk.pend;
    out->pool_checkpoints = pk.checkpoints;
    out->total_static = pc.fixed.fixed() + groups;
    out->total_pooled = pc.fixed.fixed() + pk.total;
    out->pooled = N > 1 && (cfg->flags & RP_RT_POOLED || (double)groups > 0.6 * (double)hbm_bytes);
    return RP_OK;
  } catch (const RtError& e) {
    return e.code;
  } catch (const roundpipe::InfeasibleError&) {
    return RP_E_INFEASIBLE;
  } catch (const std::exception&) {
    return RP_E_INPUT;
  }
}
