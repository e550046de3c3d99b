#pragma once
// roundpipe-b200 planner API — asymmetric stage partitioning.
//
// API-compatible with the reference partitioner
// (reference: proj/include/roundpipe/partitioner.hpp:20-276). The search is
// the paper's: every contiguous fwd/bwd time sum is a candidate t_max, each
// candidate is packed greedily (fused stage from the back, then forward
// stages left-to-right, then backward stages right-to-left), and the plan
// minimising (M*S + N*(N-1)) * t_max wins with ties broken by fewer slots
// then smaller t_max. This implementation answers every range query from
// prefix sums (the reference re-sums each range), so a pack is O(L) and the
// whole search O(L^3); results are identical, which tests/ pins against the
// reference built from source.

#include <algorithm>
#include <cstdint>
#include <limits>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <tuple>
#include <vector>

#include "roundpipe/cost_model.hpp"

namespace roundpipe {

struct InfeasibleError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Inclusive 0-based layer range; empty when last < first.
struct LayerRange {
  int first = 0;
  int last = -1;
  int size() const { return last < first ? 0 : last - first + 1; }
  bool operator==(const LayerRange&) const = default;
};

enum class StageKind { Forward, Backward, Fused };

struct StagePlan {
  std::vector<LayerRange> fwd_stages;  // ascending
  LayerRange fused_stage;              // last layers
  std::vector<LayerRange> bwd_stages;  // descending
  std::int64_t t_max_ns = 0;
  std::int64_t objective = 0;

  int s_f() const { return static_cast<int>(fwd_stages.size()); }
  int s_b() const { return 1 + static_cast<int>(bwd_stages.size()); }
  int num_slots() const { return s_f() + s_b(); }
};

struct PartitionProblem {
  std::vector<LayerCost> costs;
  int num_gpus = 1;
  int micro_batches = 1;
  std::int64_t mem_limit_bytes = std::numeric_limits<std::int64_t>::max();
  double residency_factor = 2.0;

  int num_layers() const { return static_cast<int>(costs.size()); }
  void validate() const {
    if (num_gpus < 1 || micro_batches < num_gpus || costs.empty())
      throw std::invalid_argument(
          "PartitionProblem: need N >= 1, M >= N, L >= 1");
  }
};

namespace partitioner {

namespace detail {

// Prefix sums over the cost table: every stage query becomes O(1).
struct Prefix {
  std::vector<std::int64_t> fwd, bwd, par;
  explicit Prefix(const std::vector<LayerCost>& c)
      : fwd(c.size() + 1, 0), bwd(c.size() + 1, 0), par(c.size() + 1, 0) {
    for (std::size_t i = 0; i < c.size(); ++i) {
      fwd[i + 1] = fwd[i] + c[i].t_fwd_ns;
      bwd[i + 1] = bwd[i] + c[i].t_bwd_ns;
      par[i + 1] = par[i] + c[i].param_bytes;
    }
  }
  std::int64_t time(StageKind k, int a, int b) const {  // inclusive [a, b]
    if (b < a) return 0;
    const auto& v = k == StageKind::Forward ? fwd : bwd;
    return v[b + 1] - v[a];
  }
  std::int64_t params(int a, int b) const {
    return b < a ? 0 : par[b + 1] - par[a];
  }
};

inline double footprint(StageKind k, std::int64_t params, double residency) {
  const double mult = k == StageKind::Forward ? 1.0 : 2.0;
  return residency * mult * static_cast<double>(params);
}

inline bool fits(const Prefix& px, const PartitionProblem& p, StageKind k,
                 int a, int b, std::int64_t t_max) {
  return px.time(k, a, b) <= t_max &&
         footprint(k, px.params(a, b), p.residency_factor) <=
             static_cast<double>(p.mem_limit_bytes);
}

// Greedy packing at one t_max using precomputed prefix sums.
inline std::optional<StagePlan> pack(const Prefix& px,
                                     const PartitionProblem& p,
                                     std::int64_t t_max) {
  const int L = p.num_layers();
  // fused stage: longest suffix that fits as a backward-kind stage
  int head = L;  // first layer of the fused stage
  while (head > 0 && fits(px, p, StageKind::Fused, head - 1, L - 1, t_max))
    --head;
  if (head == L) return std::nullopt;
  StagePlan plan;
  plan.fused_stage = LayerRange{head, L - 1};
  const int rem = head;  // layers [0, rem) go to fwd and bwd stages

  for (int a = 0; a < rem;) {  // forward segments, maximal from the left
    if (!fits(px, p, StageKind::Forward, a, a, t_max)) return std::nullopt;
    int b = a;
    while (b + 1 < rem && fits(px, p, StageKind::Forward, a, b + 1, t_max)) ++b;
    plan.fwd_stages.push_back(LayerRange{a, b});
    a = b + 1;
  }
  for (int b = rem - 1; b >= 0;) {  // backward segments, maximal from the right
    if (!fits(px, p, StageKind::Backward, b, b, t_max)) return std::nullopt;
    int a = b;
    while (a - 1 >= 0 && fits(px, p, StageKind::Backward, a - 1, b, t_max)) --a;
    plan.bwd_stages.push_back(LayerRange{a, b});
    b = a - 1;
  }

  std::int64_t achieved = px.time(StageKind::Fused, head, L - 1);
  for (const auto& r : plan.fwd_stages)
    achieved = std::max(achieved, px.time(StageKind::Forward, r.first, r.last));
  for (const auto& r : plan.bwd_stages)
    achieved = std::max(achieved, px.time(StageKind::Backward, r.first, r.last));
  plan.t_max_ns = achieved;
  const std::int64_t weight =
      static_cast<std::int64_t>(p.micro_batches) * plan.num_slots() +
      static_cast<std::int64_t>(p.num_gpus) * (p.num_gpus - 1);
  plan.objective = weight * achieved;
  return plan;
}

}  // namespace detail

// Per-micro-batch time of a stage (reference: partitioner.hpp:63-69).
inline std::int64_t stage_time(StageKind kind, LayerRange r,
                               const std::vector<LayerCost>& costs) {
  std::int64_t t = 0;
  for (int i = r.first; i <= r.last; ++i)
    t += kind == StageKind::Forward ? costs[i].t_fwd_ns : costs[i].t_bwd_ns;
  return t;
}

// Resident bytes of a stage: weights (fwd) or weights + grads (bwd/fused),
// times the residency factor (reference: partitioner.hpp:74-80).
inline double stage_mem_bytes(StageKind kind, LayerRange r,
                              const PartitionProblem& p) {
  std::int64_t params = 0;
  for (int i = r.first; i <= r.last; ++i) params += p.costs[i].param_bytes;
  return detail::footprint(kind, params, p.residency_factor);
}

// Sorted, de-duplicated set of all contiguous fwd and bwd time sums
// (reference: partitioner.hpp:84-101).
inline std::vector<std::int64_t> candidate_tmax(
    const std::vector<LayerCost>& costs) {
  const detail::Prefix px(costs);
  const int n = static_cast<int>(costs.size());
  std::vector<std::int64_t> out;
  out.reserve(static_cast<std::size_t>(n) * (n + 1));
  for (int a = 0; a < n; ++a)
    for (int b = a; b < n; ++b) {
      out.push_back(px.time(StageKind::Forward, a, b));
      out.push_back(px.time(StageKind::Backward, a, b));
    }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

inline bool stage_fits(StageKind kind, LayerRange r, std::int64_t t_max,
                       const PartitionProblem& p) {
  return stage_time(kind, r, p.costs) <= t_max &&
         stage_mem_bytes(kind, r, p) <= static_cast<double>(p.mem_limit_bytes);
}

// Greedy pack at a fixed t_max (reference: partitioner.hpp:113-164).
inline std::optional<StagePlan> greedy_pack(const PartitionProblem& p,
                                            std::int64_t t_max) {
  p.validate();
  if (t_max <= 0) throw std::invalid_argument("greedy_pack: t_max <= 0");
  return detail::pack(detail::Prefix(p.costs), p, t_max);
}

// Structural checks on a returned plan (reference: partitioner.hpp:167-194).
inline void validate_plan(const StagePlan& plan, const PartitionProblem& p) {
  const int L = p.num_layers();
  auto tiles = [L](const std::vector<LayerRange>& ranges,
                   const LayerRange& extra) {
    std::vector<char> hit(static_cast<std::size_t>(L), 0);
    auto mark = [&](const LayerRange& r) {
      for (int i = r.first; i <= r.last; ++i) {
        if (i < 0 || i >= L || hit[i])
          throw std::logic_error("StagePlan: ranges do not tile [0..L)");
        hit[i] = 1;
      }
    };
    for (const auto& r : ranges) mark(r);
    mark(extra);
    for (char h : hit)
      if (!h) throw std::logic_error("StagePlan: uncovered layer");
  };
  tiles(plan.fwd_stages, plan.fused_stage);
  tiles(plan.bwd_stages, plan.fused_stage);
  if (plan.fused_stage.size() < 1)
    throw std::logic_error("StagePlan: fused stage empty");
  for (const auto& r : plan.fwd_stages)
    if (stage_time(StageKind::Forward, r, p.costs) > plan.t_max_ns)
      throw std::logic_error("StagePlan: forward stage exceeds t_max");
  for (const auto& r : plan.bwd_stages)
    if (stage_time(StageKind::Backward, r, p.costs) > plan.t_max_ns)
      throw std::logic_error("StagePlan: backward stage exceeds t_max");
}

// Exhaustive candidate scan (reference: partitioner.hpp:199-216).
inline StagePlan optimal_partition(const PartitionProblem& p) {
  p.validate();
  const detail::Prefix px(p.costs);
  std::optional<StagePlan> best;
  auto key = [](const StagePlan& s) {
    return std::make_tuple(s.objective, s.num_slots(), s.t_max_ns);
  };
  for (std::int64_t t : candidate_tmax(p.costs)) {
    if (t <= 0) continue;
    auto plan = detail::pack(px, p, t);
    if (plan && (!best || key(*plan) < key(*best))) best = std::move(plan);
  }
  if (!best) throw InfeasibleError("no feasible partition at any t_max");
  validate_plan(*best, p);
  return *best;
}

// Min-max contiguous split into exactly S stages by t_fwd + t_bwd, used by
// the fixed-placement baselines (reference: partitioner.hpp:220-276).
inline std::vector<LayerRange> symmetric_split(
    const std::vector<LayerCost>& costs, int num_stages) {
  const int L = static_cast<int>(costs.size());
  if (num_stages < 1 || num_stages > L)
    throw std::invalid_argument("symmetric_split: need 1 <= S <= L");
  std::vector<std::int64_t> w(static_cast<std::size_t>(L));
  for (int i = 0; i < L; ++i) w[i] = costs[i].t_fwd_ns + costs[i].t_bwd_ns;
  // number of greedy segments at capacity `cap` (L+1 if a layer exceeds it)
  auto segments = [&](std::int64_t cap) {
    int count = 1;
    std::int64_t run = 0;
    for (std::int64_t x : w) {
      if (x > cap) return L + 1;
      if (run + x > cap) { ++count; run = 0; }
      run += x;
    }
    return count;
  };
  std::int64_t lo = *std::max_element(w.begin(), w.end());
  std::int64_t hi = std::accumulate(w.begin(), w.end(), std::int64_t{0});
  while (lo < hi) {
    const std::int64_t mid = lo + (hi - lo) / 2;
    if (segments(mid) <= num_stages) hi = mid; else lo = mid + 1;
  }
  std::vector<LayerRange> out;
  int begin = 0;
  std::int64_t run = 0;
  for (int i = 0; i < L; ++i) {
    if (run + w[i] > lo) {
      out.push_back(LayerRange{begin, i - 1});
      begin = i;
      run = 0;
    }
    run += w[i];
  }
  out.push_back(LayerRange{begin, L - 1});
  // split the widest stage (first on ties) until S stages exist
  while (static_cast<int>(out.size()) < num_stages) {
    std::size_t widest = 0;
    for (std::size_t i = 1; i < out.size(); ++i)
      if (out[i].size() > out[widest].size()) widest = i;
    if (out[widest].size() < 2) break;
    const LayerRange r = out[widest];
    const int mid = (r.first + r.last) / 2;
    out[widest] = LayerRange{r.first, mid};
    out.insert(out.begin() + static_cast<std::ptrdiff_t>(widest) + 1,
               LayerRange{mid + 1, r.last});
  }
  return out;
}

}  // namespace partitioner
}  // namespace roundpipe
