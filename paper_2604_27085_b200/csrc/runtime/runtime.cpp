// roundpipe-b200 executor: runs the RoundPipe training step on B200s.
//
// Control plane: the planner API of this repo (include/roundpipe, the
// reference's API) — optimal_partition -> slot_table_from_plan ->
// synthesize (round-robin dispatch list, reference scheduler.hpp:120-144).
// The controller walks Schedule.tasks in emission order; every (round, slot)
// runs the slot's layers for M_R micro-batches on worker task.gpu, so the
// stage->GPU assignment and execution order are the reference's by
// construction (tests compare the measured timeline's task list with the
// reference dispatcher's).
//
// Data plane, per worker, all asynchronous on CUDA streams; ONE controller
// thread enqueues everything (the paper's single controller,
// PAPER.md:352-361) in a topological order of the dependency graph:
//   compute  (high priority)  stage kernels: tcgen05 GEMMs, flash attention,
//                             fused norm/rope/swiglu, chunked LM-head + CE
//   act      (high priority)  activation/gradient hand-off, checkpoints
//   w_h2d    (low priority)   weight uploads from the pinned bf16 master
//   opt_h2d / opt_comp / opt_d2h (low priority)  AdamW on streamed fp32
//                             (master, m, v) chunks, written back to host
// The optimizer hand-off is the reference's EventPerLayer protocol
// (consistency.hpp:122-135), per layer l and iteration t:
//   (1) upload(l,t)    -> p_copy(l,t)     (2) p_copy(l,t) -> upload(l,t+1)
//   (3) GradWrite(l,t) -> g_copy(l,t)     (4) g_copy(l,t) -> GradWrite(l,t+1)
// with one cudaEvent per (action, group). g_copy(l,t) is the AdamW pass that
// consumes grad[t%2]; its bf16 result waits in `pend` until p_copy(l,t+1)
// (async, staleness 1) or is copied back at once (sync).
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <deque>
#include <unordered_map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "kernels/launch_util.h"
#include "runtime/flags.h"
#include "runtime/runtime_internal.h"

namespace rp {
namespace rt {

using roundpipe::LayerRange;
using roundpipe::StageKind;

static int64_t align128(int64_t x) { return (x + 127) / 128 * 128; }

LayerLayout make_layer_layout(const Shape& s, int lora_rank) {
  LayerLayout L;
  int64_t off = 0;
  auto put = [&](Tensor& t, int64_t rows, int64_t cols) {
    t.off = off;
    t.rows = rows;
    t.cols = cols;
    off = align128(off + rows * cols);
  };
  put(L.in_norm, s.h, 1);
  put(L.qkv, s.qkvd(), s.h);
  put(L.q_norm, s.hd, 1);
  put(L.k_norm, s.hd, 1);
  put(L.o, s.h, s.qd());
  put(L.post_norm, s.h, 1);
  if (s.moe()) {
    put(L.router, s.E, s.h);
    put(L.gate_up, (int64_t)s.E * 2 * s.m, s.h);
    put(L.down, (int64_t)s.E * s.h, s.m);
  } else {
    put(L.gate_up, 2LL * s.m, s.h);
    put(L.down, s.h, s.m);
  }
  L.lora_off = off;
  if (lora_rank > 0) {
    const int r = lora_rank;
    put(L.qkv_A, r, s.h);
    put(L.qkv_B, s.qkvd(), r);
    put(L.o_A, r, s.qd());
    put(L.o_B, s.h, r);
    if (!s.moe()) {
      put(L.gu_A, r, s.h);
      put(L.gu_B, 2LL * s.m, r);
      put(L.down_A, r, s.m);
      put(L.down_B, s.h, r);
    }
  }
  L.total = off;
  return L;
}

HeadLayout make_head_layout(const Shape& s) {
  HeadLayout H;
  H.final_norm = Tensor{0, s.h, 1};
  H.lm_head = Tensor{align128(s.h), s.V, s.h};
  H.total = align128(H.lm_head.off + (int64_t)s.V * s.h);
  return H;
}

// ---- pinned host arena -------------------------------------------------------------
// One anonymous mapping carved into 2 MiB-aligned buffers; commit() first-
// touches the pages and registers every buffer with CUDA from a pool of
// threads (pinning 100+ GB from one thread costs about a minute). Each
// buffer is its own registration, so no transfer spans two of them.
class HostArena {
 public:
  static constexpr std::size_t kAlign = std::size_t(2) << 20;
  void reserve(std::size_t bytes) {
    size_ = (bytes + kAlign - 1) & ~(kAlign - 1);
    base_ = static_cast<uint8_t*>(
        mmap(nullptr, size_, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
    if (base_ == MAP_FAILED) {
      base_ = nullptr;
      throw RtError(RP_E_INTERNAL, "mmap failed for host arena");
    }
    madvise(base_, size_, MADV_HUGEPAGE);
  }
  void* take(std::size_t bytes) {
    used_ = (used_ + kAlign - 1) & ~(kAlign - 1);
    const std::size_t len = (bytes + kAlign - 1) & ~(kAlign - 1);
    if (used_ + len > size_) throw RtError(RP_E_INTERNAL, "host arena exhausted");
    void* p = base_ + used_;
    bufs_.push_back({used_, len});
    used_ += len;
    return p;
  }
  void commit() {
    // split big buffers' first-touch across threads, register each buffer once
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::atomic<std::size_t> next{0};
    std::atomic<int> err{0};
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
      th.emplace_back([&] {
        for (std::size_t i; (i = next++) < bufs_.size();) {
          std::memset(base_ + bufs_[i].first, 0, bufs_[i].second);
          if (cudaHostRegister(base_ + bufs_[i].first, bufs_[i].second,
                               cudaHostRegisterPortable) != cudaSuccess)
            err = 1;
        }
      });
    for (auto& t : th) t.join();
    registered_ = true;
    if (err) throw RtError(RP_E_CUDA, "cudaHostRegister failed");
  }
  std::size_t size() const { return size_; }
  ~HostArena() {
    if (!base_) return;
    if (registered_)
      for (const auto& b : bufs_) cudaHostUnregister(base_ + b.first);
    munmap(base_, size_);
  }

 private:
  uint8_t* base_ = nullptr;
  std::size_t size_ = 0, used_ = 0;
  std::vector<std::pair<std::size_t, std::size_t>> bufs_;
  bool registered_ = false;
};

// ---- the runtime --------------------------------------------------------------------
struct Runtime {
  rp_runtime_config_t cfg{};
  std::string model;
  Shape s;
  LayerLayout LL;
  HeadLayout HL;
  int T = 0, M = 0, MR = 0, N = 1, R = 1, S = 1, ndev = 1;
  std::vector<roundpipe::LayerCost> costs;
  roundpipe::StagePlan plan;
  std::vector<roundpipe::StageSlot> slots;
  std::vector<int> bwd_slot_of;  // decoder layer -> slot index recomputing it
  roundpipe::Schedule sched;
  int horizon = 0;
  HostArena arena;
  std::vector<HostGroup> host;       // g = group + 1
  std::vector<Gpu> gpus;             // logical workers
  std::vector<int> grad_owner;       // g -> worker holding this iteration's grads
  std::vector<int> pend_owner;       // g -> worker holding pending AdamW output (-1 none)
  // optimizer hand-off protocol state (consistency.hpp:122-135): per group
  // the ParamCopy index of the latest p_copy (-1 none) and the newest
  // iteration whose weights were uploaded; flag words: pub(g) = latest
  // published ParamCopy index + 1, loss(w) = latest iteration + 1 whose loss
  // worker w has copied to the host
  std::vector<int> pcopy_idx, upload_ver;
  FlagWords flags;
  int flag_pub(int g) const { return g; }
  int flag_loss(int w) const { return ngroups() + w; }
  // realised protocol edges (RP_RT_RECORD_PROTOCOL): (kind, group, iteration)
  // of the action waited on -> of the waiting action
  struct ProtoEdge {
    int bk, bg, bi, ak, ag, ai;
  };
  std::vector<ProtoEdge> proto;
  void proto_edge(roundpipe::ActionKind bk, int bg, int bi, roundpipe::ActionKind ak, int ag,
                  int ai) {
    if ((cfg.flags & RP_RT_RECORD_PROTOCOL) && bi >= 0)
      proto.push_back({(int)bk, bg, bi, (int)ak, ag, ai});
  }
  std::vector<cudaEvent_t> state_ev; // g -> event of the latest fp32 state write-back
  std::vector<std::vector<int>> uploaders;  // g -> workers that uploaded this version
  std::vector<char> fused_worker;    // worker ran a fused task this iteration
  int iter = 0, last_iter = -1;
  bool grads_pending = false;
  float* loss_host = nullptr;        // pinned [2][N] (iteration parity)
  std::vector<cudaEvent_t> ev_loss;  // per worker, after its last fused task
  // per iteration parity: which workers ran a fused slot, the loss scale, and
  // the iteration number (non-blocking forward_backward / rp_loss)
  std::vector<char> fused_par[2];
  float grad_scale_par[2] = {0.f, 0.f};
  int iter_par[2] = {-1, -1};
  void enqueue_iteration(const int32_t* tokens, const int32_t* labels);
  float wait_loss(int it);
  std::vector<TaskRecord> records;
  // transfer / optimizer intervals for the measured timeline
  struct XferRecord {
    int kind, group, iteration, worker;  // kind: 0 upload, 1 p_copy, 2 AdamW group
    cudaEvent_t a, b;
  };
  std::vector<XferRecord> xfers;
  bool tl_on() const { return cfg.flags & RP_RT_RECORD_TIMELINE; }
  cudaEvent_t xfer_begin(cudaStream_t st) {
    if (!tl_on()) return nullptr;
    cudaEvent_t e = new_event(true);
    RP_CUDA(cudaEventRecord(e, st));
    return e;
  }
  void xfer_end(cudaEvent_t a, cudaStream_t st, int kind, int g, int it, int w) {
    if (!a) return;
    cudaEvent_t e = new_event(true);
    RP_CUDA(cudaEventRecord(e, st));
    xfers.push_back({kind, g, it, w, a, e});
  }
  std::vector<cudaEvent_t> event_pool;
  int64_t h2d_bytes = 0, d2h_bytes = 0, p2p_bytes = 0, kernels = 0;
  int64_t chunk_elems = 32ll << 20;  // optimizer chunk (elements)
  int logits_rows = 2048;            // LM-head chunk rows (2 chunks per 4K micro-batch)
  int parities = 1;                  // hand-off / checkpoint buffer sets
  // kernel profiling (one step at a time): per category CUDA-event pairs
  // around each launch on its own stream, with the launch's algorithmic work
  struct ProfRec {
    int cat;
    cudaEvent_t a, b;
    double work;
    int worker, lane;  // lane 0 = compute stream, 1 = optimizer stream
    int unit, inst;    // (layer, phase) being executed and its call instance
  };
  // current compute unit for the profile records: layer l (L = head) and
  // phase (0 fwd, 1 bwd, 2 recompute fwd, 3 head fwd+bwd), one instance per call
  int prof_layer = -1, prof_phase = 0, prof_inst = 0;
  void prof_unit(int layer, int phase) {
    prof_layer = layer;
    prof_phase = phase;
    ++prof_inst;
  }
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> prof_pool;
  std::size_t prof_next = 0;
  cudaEvent_t prof_event() {
    if (prof_next == prof_pool.size()) prof_pool.push_back(new_event(true));
    return prof_pool[prof_next++];
  }
  int prof_begin(cudaStream_t st) {
    if (!prof_on) return -1;
    ProfRec r{0, prof_event(), prof_event(), 0.0, 0, 0, prof_layer * 4 + prof_phase, prof_inst};
    for (const Gpu& G : gpus)
      if (G.compute == st || G.opt_comp == st || G.opt_res == st || G.wgrad == st ||
          G.fwd2 == st) {
        r.worker = G.id;
        r.lane = (G.opt_comp == st || G.opt_res == st) ? 1 : (G.wgrad == st ? 2 : 0);
      }
    RP_CUDA(cudaEventRecord(r.a, st));
    prof.push_back(r);
    return (int)prof.size() - 1;
  }
  void prof_end(int idx, cudaStream_t st, int cat, double work) {
    if (idx < 0) return;
    prof[idx].cat = cat;
    prof[idx].work = work;
    RP_CUDA(cudaEventRecord(prof[idx].b, st));
  }

  int ngroups() const { return s.L + 2; }
  // device bytes of one worker's per-group buffers without pooling: two bf16
  // weight versions, two fp32 grad buffers, the AdamW output, checkpoints
  std::size_t static_bytes_per_worker() const {
    std::size_t b = 0;
    for (int g = 0; g < ngroups(); ++g)
      b += (std::size_t)host[g].n * 2 * 3 + (std::size_t)host[g].tn() * 4 * 2;
    const int lck = std::max(0, plan.fused_stage.first);
    if (S > 1) b += (std::size_t)parities * lck * MR * T * s.h * 2;
    return b;
  }
  int64_t group_numel(int g) const {
    if (g == 0) return (int64_t)s.V * s.h;
    if (g == s.L + 1) return HL.total;
    return LL.total;
  }
  int worker_of(int round, int slot) const { return (int)(((int64_t)round * S + slot) % N); }

  void init(const rp_runtime_config_t& c);
  void build_plan();
  void ensure_horizon(int it);
  void alloc_worker(Gpu& G, int id);
  void init_weights();
  cudaEvent_t new_event(bool timing);
  void set_dev(const Gpu& G) { RP_CUDA(cudaSetDevice(G.dev)); }
  // device memory of worker G (current device = G.dev), tracked for ~Runtime
  void* dalloc(Gpu& G, std::size_t bytes, int cat) {
    void* p = nullptr;
    RP_CUDA(cudaMalloc(&p, std::max<std::size_t>(bytes, 256)));
    G.allocated[cat] += bytes;
    G.owned.push_back(p);
    return p;
  }
  void dfree(Gpu& G, void* p) {
    auto it = std::find(G.owned.begin(), G.owned.end(), p);
    if (it == G.owned.end()) throw RtError(RP_E_INTERNAL, "freeing an untracked device buffer");
    G.owned.erase(it);
    RP_CUDA(cudaFree(p));
  }
  // stream `to` waits for everything enqueued on `from` so far (both on
  // worker G's device); the fork events are reused round-robin (a wait
  // captures the event's state when it is enqueued)
  void join(Gpu& G, cudaStream_t from, cudaStream_t to) {
    cudaEvent_t& e = G.fork_ev[G.fork_i++ & 63];
    if (!e) e = new_event(false);
    RP_CUDA(cudaEventRecord(e, from));
    RP_CUDA(cudaStreamWaitEvent(to, e, 0));
  }
  // ---- per-worker buffer pools (N > 1: "stateless" workers) -------------------
  // A worker holds weights only for the versions it is about to use or using,
  // grads only until the optimizer consumed them, AdamW output until p_copy,
  // checkpoints until the recomputing slot read them — so its HBM footprint
  // is its working set, not the model (a Qwen3-32B at N=8 would need ~0.4 TB
  // per worker with one buffer per group). Slabs are exact-size, allocated
  // on first need and reused through their free events.
  bool pooled = false;
  int slab_acquire(Gpu& G, std::size_t bytes, int cat, cudaStream_t user) {
    int cur = 0;
    RP_CUDA(cudaGetDevice(&cur));
    RP_CUDA(cudaSetDevice(G.dev));
    int idx = -1;
    for (int i = 0; i < (int)G.slabs.size(); ++i)
      if (!G.slabs[i].busy && G.slabs[i].bytes == bytes) {
        idx = i;
        break;
      }
    if (idx < 0) {
      Slab sl;
      sl.bytes = bytes;
      sl.p = dalloc(G, bytes, cat);
      sl.free_ev = new_event(false);
      G.slabs.push_back(sl);
      G.pool_bytes += bytes;
      idx = (int)G.slabs.size() - 1;
    }
    Slab& sl = G.slabs[idx];
    if (sl.recorded) RP_CUDA(cudaStreamWaitEvent(user, sl.free_ev, 0));  // previous user done
    sl.busy = true;
    sl.cat = cat;
    G.pool_busy += bytes;
    G.pool_peak = std::max(G.pool_peak, G.pool_busy);
    RP_CUDA(cudaSetDevice(cur));
    return idx;
  }
  // the slab's last access was enqueued on `st` (a stream of G's device)
  void slab_release(Gpu& G, int idx, cudaStream_t st, int tag_kind = -1, int tag_group = -1,
                    int tag_iter = -1) {
    Slab& sl = G.slabs.at(idx);
    if (!sl.busy) throw RtError(RP_E_INTERNAL, "releasing a free slab");
    int cur = 0;
    RP_CUDA(cudaGetDevice(&cur));
    RP_CUDA(cudaSetDevice(G.dev));
    RP_CUDA(cudaEventRecord(sl.free_ev, st));
    RP_CUDA(cudaSetDevice(cur));
    sl.recorded = true;
    sl.busy = false;
    sl.tag_kind = tag_kind;
    sl.tag_group = tag_group;
    sl.tag_iter = tag_iter;
    G.pool_busy -= sl.bytes;
  }
  // (worker, group) -> (round, slot) of its last use in the iteration being enqueued
  std::unordered_map<int64_t, int64_t> last_use_task;
  // producer P finished writing hand-off / checkpoint buffer b on stream st
  void mark_ready(Slotbuf& b, const Gpu& P, cudaStream_t st) {
    cudaEvent_t& e = b.ready_dev[P.dev];
    if (!e) e = new_event(false);  // created on the producer's device (current)
    RP_CUDA(cudaEventRecord(e, st));
    b.ready = e;
  }
  void d2d(void* dst, const Gpu& Gd, const void* src, const Gpu& Gs, std::size_t bytes,
           cudaStream_t st);

  void forward_backward(const int32_t* tokens, const int32_t* labels, float* loss);
  void run_slot(Gpu& G, int it, int round, int slot, int first_round, float grad_scale);
  void upload(Gpu& G, int g, int it, bool last_use);
  bool upload_reserve(Gpu& G, int g, int it);
  void upload_chunk(Gpu& G, int g, int it, int64_t off, int64_t len);
  void upload_done(Gpu& G, int g, int it);
  void prefetch(int it, bool reverse = false);
  // LPT-windowed uploads of the next iteration (async), released one window
  // per micro-batch start of the worker's compute
  struct UpChunk {
    int g;
    int64_t off, len;  // bytes within the group's bf16 buffer
  };
  struct UpWindow {
    int it = 0;
    std::vector<UpChunk> chunks;
  };
  std::vector<std::deque<UpWindow>> upq;   // per worker
  std::vector<std::vector<int>> up_left;   // per worker, per group: chunks not yet enqueued
  void plan_upload_windows(int it_next);
  void release_window(Gpu& G);
  void flush_windows();
  std::vector<int> slot_groups(const roundpipe::StageSlot& ss) const;
  int exec_iter = 0;  // iteration whose compute is being enqueued
  void p_copy(int g);
  void layer_fwd(Gpu& G, int l, const uint16_t* x, LayerActs& A, uint16_t* x_out,
                 cudaStream_t on = nullptr);
  void layer_bwd(Gpu& G, int l, LayerActs& A, bool first);
  void head_fwd_bwd(Gpu& G, const uint16_t* x, int gmb, bool first, float grad_scale,
                    cudaStream_t on = nullptr);
  void step();
  void adam_group(Gpu& G, int g, int parity);
  void place_resident_state();      // choose groups whose fp32 state lives in HBM
  void publish_in_place();          // one worker: streamed groups publish into w[] too
  void push_resident(int g);        // host master/m/v -> device state
  void pull_resident(int g);        // device state -> host master/m/v (if stale)
  void pull_w16(int g);             // direct groups: device bf16 of the next iteration -> host
  int64_t resident_params = 0;
  int lora_r = 0;          // LoRA rank (0 = full fine-tune)
  int64_t partition_limit = 0;  // memory limit the partitioner planned with
  float lora_scale = 0.f;  // alpha / r
  bool trainable(int g) const { return host[g].tn() > 0; }
  // LoRA: Y += s (X A^T) B^T; keeps Us = s X A^T (T x r) for the backward
  // One linear layer's forward, Y = X W^T (+ R). LoRA: Us = s X A^T first, then
  // Y = X W^T + Us B^T (+ R) as ONE GEMM with a second K segment (no rank-r
  // update pass over Y).
  void lin_fwd(cudaStream_t st, const uint16_t* W, const Tensor& Tw, const Tensor* Ta,
               const Tensor* Tb, const uint16_t* X, int64_t ldx, int in, uint16_t* Us,
               uint16_t* Y, int64_t ldy, int out, const void* R = nullptr, int64_t ldr = 0) {
    if (!lora_r) {
      gemm(st, X, ldx, false, W + Tw.off, in, false, Y, ldy, false, false, T, out, in, R, ldr);
      return;
    }
    const int r = lora_r;
    gemm(st, X, ldx, false, W + Ta->off, in, false, Us, r, false, false, T, r, in);
    RP_K(rp_scale_bf16(Us, (int64_t)T * r, lora_scale, st));
    gemm2(st, X, ldx, false, W + Tw.off, in, false, Y, ldy, T, out, in, R, ldr, Us, r,
          W + Tb->off, r, r);
    kernels += 1;
  }
  // One linear layer's input gradient, dX = dY W. LoRA: dUs = s dY B first,
  // then dX = dY W + dUs A as one two-segment GEMM; lora_wgrad() afterwards.
  void lin_dgrad(Gpu& G, cudaStream_t st, const uint16_t* W, const Tensor& Tw, const Tensor* Ta,
                 const Tensor* Tb, const uint16_t* dY, int64_t ldy, int out, uint16_t* dX,
                 int64_t lddx, int in, bool swiglu_bwd = false, const void* gu = nullptr) {
    if (!lora_r) {
      gemm(st, dY, ldy, false, W + Tw.off, in, true, dX, lddx, false, false, T, in, out,
           swiglu_bwd ? gu : nullptr, swiglu_bwd ? lddx : 0, swiglu_bwd);
      return;
    }
    const int r = lora_r;
    gemm(st, dY, ldy, false, W + Tb->off, r, true, G.du, r, false, false, T, r, out);
    RP_K(rp_scale_bf16(G.du, (int64_t)T * r, lora_scale, st));
    gemm2(st, dY, ldy, false, W + Tw.off, in, true, dX, lddx, T, in, out, nullptr, 0, G.du, r,
          W + Ta->off, in, r);
    kernels += 1;
  }
  // LoRA adapter gradients of one linear (after lin_dgrad): dB += dY^T Us,
  // dA += dUs^T X
  void lora_wgrad(Gpu& G, cudaStream_t st, float* dW, const Tensor& Ta, const Tensor& Tb,
                  const uint16_t* X, int64_t ldx, int in, const uint16_t* Us, const uint16_t* dY,
                  int64_t ldy, int out, bool first) {
    const int r = lora_r;
    gemm(st, dY, ldy, true, Us, r, true, dW + Tb.off, r, true, !first, out, r, T);
    gemm(st, G.du, r, true, X, ldx, true, dW + Ta.off, in, true, !first, r, in, T);
  }
  // before the first grad write of an HBM-resident group g in an iteration:
  // AdamW of the previous iteration has consumed its single grad buffer (edge 4)
  // (the latest AdamW on this worker's buffer: resident AdamW passes of a
  // group are chained through state_ev, so it implies every earlier one)
  void grad_free(Gpu& G, int g, cudaStream_t q) {
    if (!host[g].d_state) return;  // streamed groups: two buffers, waited at slot start
    DevGroup& D = G.groups[g];
    const int p = D.adam_iter[0] >= D.adam_iter[1] ? 0 : 1;
    if (D.adam_iter[p] < 0) return;
    RP_CUDA(cudaStreamWaitEvent(q, D.ev_adam[p], 0));  // edge (4)
    proto_edge(roundpipe::ActionKind::GradCopy, g, D.adam_iter[p],
               roundpipe::ActionKind::GradWrite, g, exec_iter);
  }
  void sync_all();
  void gemm(cudaStream_t st, const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb,
            bool b_mn, void* D, int64_t ldd, bool f32, bool acc, int M_, int N_, int K_,
            const void* Rz = nullptr, int64_t ldr = 0, bool swiglu_bwd = false);
  void gemm2(cudaStream_t st, const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb,
             bool b_mn, void* D, int64_t ldd, int M_, int N_, int K_, const void* Rz, int64_t ldr,
             const void* A2, int64_t lda2, const void* B2, int64_t ldb2, int K2);
  // grouped expert GEMM over the expert-sorted rows (row offsets on the device)
  void grouped(cudaStream_t st, const void* A, int64_t lda, const void* B, int64_t ldb, bool b_mn,
               void* D, int64_t ldd, int M_, int N_, int K_, const int32_t* off, int brows,
               const void* gu = nullptr) {
    rp_gemm_args_t a{};
    a.M = M_;
    a.N = N_;
    a.K = K_;
    a.A = A;
    a.lda = lda;
    a.B = B;
    a.ldb = ldb;
    a.b_mn_major = b_mn;
    a.D = D;
    a.ldd = ldd;
    a.R = gu;
    a.ldr = gu ? 2LL * N_ : 0;
    const int pi = prof_begin(st);
    RP_K(rp_gemm_grouped(&a, off, s.E, brows, gu ? 1 : 0, st));
    prof_end(pi, st, 0, 2.0 * M_ * N_ * (double)K_);
    ++kernels;
  }
  void moe_mlp_fwd(Gpu& G, cudaStream_t st, const uint16_t* W, LayerActs& A, uint16_t* x_out);
  void moe_mlp_bwd(Gpu& G, cudaStream_t st, const uint16_t* W, LayerActs& A, const uint16_t* dy,
                   uint16_t* dgu);
  ~Runtime();
};

cudaEvent_t Runtime::new_event(bool timing) {
  cudaEvent_t e;
  RP_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  event_pool.push_back(e);
  return e;
}

void Runtime::d2d(void* dst, const Gpu& Gd, const void* src, const Gpu& Gs, std::size_t bytes,
                  cudaStream_t st) {
  if (Gd.dev == Gs.dev) {
    RP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
  } else {  // NVLink peer copy through NVSwitch
    RP_CUDA(cudaMemcpyPeerAsync(dst, Gd.dev, src, Gs.dev, bytes, st));
    p2p_bytes += (int64_t)bytes;
  }
}

void Runtime::gemm(cudaStream_t st, const void* A, int64_t lda, bool a_mn, const void* B,
                   int64_t ldb, bool b_mn, void* D, int64_t ldd, bool f32, bool acc, int M_,
                   int N_, int K_, const void* Rz, int64_t ldr, bool swiglu_bwd) {
  rp_gemm_args_t a{};
  a.M = M_;
  a.N = N_;
  a.K = K_;
  a.A = A;
  a.lda = lda;
  a.a_mn_major = a_mn;
  a.B = B;
  a.ldb = ldb;
  a.b_mn_major = b_mn;
  a.D = D;
  a.ldd = ldd;
  a.out_f32 = f32;
  a.accumulate = acc;
  a.R = Rz;
  a.ldr = ldr;
  const int pi = prof_begin(st);
  const int rc = swiglu_bwd ? rp_gemm_swiglu_bwd(&a, st) : rp_gemm_bf16(&a, st);
  if (rc != RP_OK)
    throw RtError(rc, "gemm failed: M " + std::to_string(M_) + " N " + std::to_string(N_) + " K " +
                          std::to_string(K_) + " lda " + std::to_string(lda) + " ldb " +
                          std::to_string(ldb) + " ldd " + std::to_string(ldd) + " a_mn " +
                          std::to_string(a_mn) + " b_mn " + std::to_string(b_mn) + " f32 " +
                          std::to_string(f32) + " acc " + std::to_string(acc) + " R " +
                          std::to_string(Rz != nullptr) + " swiglu_bwd " +
                          std::to_string(swiglu_bwd) + " -> " + rp_gemm_last_error() + " / " +
                          cudaGetErrorString(cudaGetLastError()));
  prof_end(pi, st, 0, 2.0 * M_ * N_ * (double)K_);
  ++kernels;
}

void Runtime::gemm2(cudaStream_t st, const void* A, int64_t lda, bool a_mn, const void* B,
                    int64_t ldb, bool b_mn, void* D, int64_t ldd, int M_, int N_, int K_,
                    const void* Rz, int64_t ldr, const void* A2, int64_t lda2, const void* B2,
                    int64_t ldb2, int K2) {
  rp_gemm_args_t a{};
  a.M = M_;
  a.N = N_;
  a.K = K_;
  a.A = A;
  a.lda = lda;
  a.a_mn_major = a_mn;
  a.B = B;
  a.ldb = ldb;
  a.b_mn_major = b_mn;
  a.D = D;
  a.ldd = ldd;
  a.R = Rz;
  a.ldr = ldr;
  const int pi = prof_begin(st);
  RP_K(rp_gemm_bf16_2seg(&a, A2, lda2, B2, ldb2, K2, st));
  prof_end(pi, st, 0, 2.0 * M_ * N_ * (double)(K_ + K2));
  ++kernels;
}

void Runtime::init(const rp_runtime_config_t& c) {
  cfg = c;
  model = c.model ? c.model : "qwen3-8b";
  cfg.model = nullptr;
  s = load_shape(model);
  if (c.seq_len < 128 || c.seq_len % 128 || c.micro_batch < 1 || c.micro_batches < 1 ||
      c.num_gpus < 1)
    throw RtError(RP_E_INPUT, "need seq_len % 128 == 0, b >= 1, M >= 1, N >= 1");
  if (s.h % 64 || s.m % 64 || (s.hd != 64 && s.hd != 128) || s.V % 8 || s.nq % s.nk)
    throw RtError(RP_E_INPUT, "unsupported model dims");
  T = c.seq_len * c.micro_batch;
  M = c.micro_batches;
  N = c.num_gpus;
  RP_CUDA(cudaGetDeviceCount(&ndev));
  if (ndev < 1) throw RtError(RP_E_CUDA, "no CUDA device");
  ndev = std::min(ndev, N);
  for (int a = 0; a < ndev; ++a)  // NVLink P2P for hand-offs between workers
    for (int b = 0; b < ndev; ++b) {
      int ok = 0;
      if (a == b || cudaDeviceCanAccessPeer(&ok, a, b) != cudaSuccess || !ok) continue;
      RP_CUDA(cudaSetDevice(a));
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) RP_CUDA(e);
      cudaGetLastError();
    }
  if (cfg.lora_rank < 0 || cfg.lora_rank > 256 || cfg.lora_rank % 8)
    throw RtError(RP_E_INPUT, "lora_rank must be 0 or a multiple of 8 up to 256");
  if (s.moe() && cfg.lora_rank == 0)  // BASELINE configs[4]: LoRA of a frozen MoE base
    throw RtError(RP_E_INPUT, "MoE models: LoRA fine-tune only (experts and router frozen)");
  lora_r = cfg.lora_rank;
  lora_scale = lora_r > 0 ? (cfg.lora_alpha > 0 ? cfg.lora_alpha : (float)lora_r) / lora_r : 0.f;
  LL = make_layer_layout(s, lora_r);
  HL = make_head_layout(s);
  if (cfg.logits_rows) {  // LM-head chunk rows
    if (cfg.logits_rows < 128 || cfg.logits_rows % 128)
      throw RtError(RP_E_INPUT, "logits_rows must be a positive multiple of 128");
    logits_rows = cfg.logits_rows;
  }
  if (!(cfg.residency_factor > 0)) cfg.residency_factor = 2.0;
  if (cfg.adam.lr == 0.f && cfg.adam.beta1 == 0.f) {
    cfg.adam = rp_adam_hparams_t{1e-4f, 0.9f, 0.95f, 1e-8f, 0.0f, 1.0f};
  }
  if (cfg.adam.grad_scale == 0.f) cfg.adam.grad_scale = 1.f;
  build_plan();
  MR = c.round_micro_batches ? c.round_micro_batches : M;
  R = M / MR;
  if (R > 1 && N > 1)
    throw RtError(RP_E_INPUT, "multi-round iterations need N == 1 (host grad merge not built)");
  parities = N > 1 ? 2 : 1;

  host.resize(ngroups());
  std::size_t bytes = 0;
  for (int g = 0; g < ngroups(); ++g) {
    HostGroup& H = host[g];
    H.n = group_numel(g);
    H.t_off = lora_r == 0 ? 0 : (g >= 1 && g <= s.L ? LL.lora_off : H.n);
    bytes += (std::size_t)H.n * 2 + (std::size_t)H.tn() * 12 + 4 * HostArena::kAlign;
  }
  arena.reserve(bytes);
  for (int g = 0; g < ngroups(); ++g) {
    HostGroup& H = host[g];
    H.w16 = static_cast<uint16_t*>(arena.take(H.n * 2));
    if (H.tn() > 0) {  // shifted: valid for global offsets >= t_off
      H.master = static_cast<float*>(arena.take(H.tn() * 4)) - H.t_off;
      H.m = static_cast<float*>(arena.take(H.tn() * 4)) - H.t_off;
      H.v = static_cast<float*>(arena.take(H.tn() * 4)) - H.t_off;
    }
  }
  arena.commit();
  grad_owner.assign(ngroups(), 0);
  pend_owner.assign(ngroups(), -1);
  pcopy_idx.assign(ngroups(), -1);
  upload_ver.assign(ngroups(), -1);
  upq.assign(N, {});
  up_left.assign(N, std::vector<int>(ngroups(), 0));
  state_ev.assign(ngroups(), nullptr);
  uploaders.assign(ngroups(), {});
  RP_CUDA(cudaMallocHost(&loss_host, sizeof(float) * N * 2));
  RP_CUDA(cudaSetDevice(0));
  flags.init(ngroups() + N);
  // pooled workers: requested, or one-buffer-per-group would not fit
  if (N > 1) {
    cudaDeviceProp prop;
    RP_CUDA(cudaGetDeviceProperties(&prop, 0));
    const int per_dev = (N + ndev - 1) / ndev;
    const double need = (double)per_dev * (double)static_bytes_per_worker();
    pooled = (cfg.flags & RP_RT_POOLED) || need > 0.6 * (double)prop.totalGlobalMem;
  }
  gpus.resize(N);
  for (int w = 0; w < N; ++w) alloc_worker(gpus[w], w);
  ev_loss.resize(N);
  for (int w = 0; w < N; ++w) {
    set_dev(gpus[w]);
    ev_loss[w] = new_event(false);
  }
  if (!(cfg.flags & RP_RT_SKIP_INIT)) init_weights();
  sync_all();
  place_resident_state();
  publish_in_place();
}

// One worker on one device: the streamed (host-offloaded) groups' AdamW
// writes its bf16 result straight into the device buffer of the version that
// will use it, as the HBM-resident groups do — the fp32 master/m/v still
// stream through the GPU every step (BASELINE configs[2]), but the bf16
// weights no longer round-trip through the pinned master (p_copy D2H +
// upload H2D: 2 x 16.4 GB of PCIe per Qwen3-8B step). Same versions, same
// staleness; the host bf16 copy is refreshed on demand (pull_w16).
// RP_RT_HOST_PUBLISH keeps the paper's p_copy / upload path.
void Runtime::publish_in_place() {
  if (N != 1 || ndev != 1 || pooled || (cfg.flags & RP_RT_HOST_PUBLISH)) return;
  Gpu& G = gpus[0];
  set_dev(G);
  for (int g = 0; g < ngroups(); ++g) {
    HostGroup& H = host[g];
    if (H.direct || H.tn() == 0) continue;
    DevGroup& D = G.groups[g];
    if (D.pend) {
      dfree(G, D.pend + H.t_off);
      D.pend = nullptr;
      G.allocated[2] -= (std::size_t)H.tn() * 2;
    }
    H.direct = true;
  }
}

// Optimizer state in free HBM (single device only: with N devices a group's
// grads land on a different device every iteration). Greedy over groups,
// largest first, until the free memory minus a reserve is used; the rest
// streams from pinned host memory. cfg.resident_state_gb: < 0 no cap, 0 off
// (every group host-offloaded: BASELINE configs[2]), > 0 cap in GB.
void Runtime::place_resident_state() {
  if (ndev != 1 || pooled) return;
  const double cap_gb = cfg.resident_state_gb < 0 ? 1e9 : cfg.resident_state_gb;
  if (cap_gb <= 0) return;
  set_dev(gpus[0]);
  std::size_t free_b = 0, total_b = 0;
  RP_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const std::size_t reserve = std::size_t(6) << 30;  // allocator, cuBLAS-free kernels, slack
  int64_t budget = (int64_t)free_b - (int64_t)reserve;  // device memory
  const int64_t cap = (int64_t)std::min(cap_gb * 1e9, 9.0e18);  // resident state bytes
  int64_t placed = 0;
  std::vector<int> order(ngroups());
  for (int g = 0; g < ngroups(); ++g) order[g] = g;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return host[a].tn() > host[b].tn(); });
  // A resident group needs 12 B/param of state but only ONE fp32 grad buffer
  // (its AdamW finishes within milliseconds of GradWrite, long before the next
  // iteration's first write of that group), so converting a group costs a net
  // 8 B/param: free grad[1] on every worker first, then allocate the state.
  for (int g : order) {
    const int64_t n = host[g].tn(), o = host[g].t_off;
    if (n == 0) continue;  // frozen group
    // publish straight into the device weights (unless asked to go through
    // the pinned bf16 master as with several workers)
    const bool direct = N == 1 && !(cfg.flags & RP_RT_HOST_PUBLISH);
    const int64_t freed = n * 4 * (int64_t)gpus.size() + (direct ? host[g].n * 2 : 0);
    if (n * 12 > budget + freed || placed + n * 12 > cap) continue;
    for (Gpu& G : gpus) {
      DevGroup& D = G.groups[g];
      dfree(G, D.grad[1] + o);
      D.grad[1] = D.grad[0];
      G.allocated[1] -= (std::size_t)n * 4;
      if (direct) {
        dfree(G, D.pend + host[g].t_off);
        D.pend = nullptr;
        G.allocated[2] -= (std::size_t)host[g].tn() * 2;
      }
    }
    host[g].direct = direct;
    budget += freed;
    void* p = nullptr;
    if (cudaMalloc(&p, (std::size_t)(n * 12)) != cudaSuccess) {
      cudaGetLastError();
      for (Gpu& G : gpus) {  // undo: back to two buffers (and a pend buffer)
        DevGroup& D = G.groups[g];
        D.grad[1] = static_cast<float*>(dalloc(G, (std::size_t)n * 4, 1)) - o;
        if (!D.pend)
          D.pend = static_cast<uint16_t*>(dalloc(G, (std::size_t)host[g].tn() * 2, 2)) - host[g].t_off;
      }
      host[g].direct = false;
      break;
    }
    host[g].d_state = static_cast<float*>(p);
    budget -= n * 12;
    placed += n * 12;
    resident_params += n;
    gpus[0].allocated[7] += (std::size_t)(n * 12);
    push_resident(g);
  }
}

void Runtime::push_resident(int g) {
  HostGroup& H = host[g];
  if (!H.d_state) return;
  set_dev(gpus[0]);
  const int64_t tn = H.tn(), o = H.t_off;
  RP_CUDA(cudaMemcpy(H.d_state, H.master + o, tn * 4, cudaMemcpyHostToDevice));
  RP_CUDA(cudaMemcpy(H.d_state + tn, H.m + o, tn * 4, cudaMemcpyHostToDevice));
  RP_CUDA(cudaMemcpy(H.d_state + 2 * tn, H.v + o, tn * 4, cudaMemcpyHostToDevice));
  H.host_stale = false;
}

void Runtime::pull_w16(int g) {
  HostGroup& H = host[g];
  if (!H.direct || !H.w16_stale) return;
  DevGroup& D = gpus[0].groups[g];
  // the version the next iteration computes with: the newest one not beyond
  // it (a pending staleness-1 update, version iter+1, is not published yet;
  // without step() calls in between, the newest version is older than iter)
  int b = -1;
  for (int c = 0; c < 2; ++c)
    if (D.loaded[c] >= 0 && D.loaded[c] <= iter && (b < 0 || D.loaded[c] > D.loaded[b])) b = c;
  if (b < 0) throw RtError(RP_E_INTERNAL, "direct group: no current weights on the device");
  set_dev(gpus[0]);
  RP_CUDA(cudaMemcpy(H.w16 + H.t_off, D.w[b] + H.t_off, H.tn() * 2, cudaMemcpyDeviceToHost));
  H.w16_stale = false;
}

void Runtime::pull_resident(int g) {
  HostGroup& H = host[g];
  if (!H.d_state || !H.host_stale) return;
  set_dev(gpus[0]);
  const int64_t tn = H.tn(), o = H.t_off;
  RP_CUDA(cudaMemcpy(H.master + o, H.d_state, tn * 4, cudaMemcpyDeviceToHost));
  RP_CUDA(cudaMemcpy(H.m + o, H.d_state + tn, tn * 4, cudaMemcpyDeviceToHost));
  RP_CUDA(cudaMemcpy(H.v + o, H.d_state + 2 * tn, tn * 4, cudaMemcpyDeviceToHost));
  H.host_stale = false;
}

void Runtime::build_plan() {
  cudaDeviceProp prop;
  RP_CUDA(cudaGetDeviceProperties(&prop, 0));
  PlanChoice pc = choose_plan(cfg, s, model, (int64_t)prop.totalGlobalMem, logits_rows, chunk_elems);
  cfg.costs = nullptr;  // the caller's table was copied
  costs = std::move(pc.costs);
  plan = pc.plan;
  slots = std::move(pc.slots);
  partition_limit = pc.mem_limit;
  S = (int)slots.size();
  bwd_slot_of.assign(s.L, -1);
  for (const auto& sl : slots)
    if (sl.kind == StageKind::Backward)
      for (int l = sl.layers.first; l <= sl.layers.last; ++l) bwd_slot_of[l] = sl.index;
  ensure_horizon(8);
}

void Runtime::ensure_horizon(int it) {
  if (it < horizon) return;
  int h = std::max(8, horizon);
  while (h <= it) h *= 2;
  roundpipe::ScheduleSpec spec;
  spec.kind = cfg.async_optimizer ? roundpipe::ScheduleKind::RoundPipe
                                  : roundpipe::ScheduleKind::RoundPipeSync;
  spec.num_gpus = cfg.num_gpus;
  spec.micro_batches = cfg.micro_batches;
  spec.round_micro_batches = cfg.round_micro_batches ? cfg.round_micro_batches : cfg.micro_batches;
  spec.iterations = h;
  for (const auto& sl : slots) spec.slot_durs.push_back(sl.dur_ns);
  sched = roundpipe::scheduler::synthesize(spec);
  if (auto err = roundpipe::scheduler::validate(sched))
    throw RtError(RP_E_INTERNAL, "dispatch list invalid: " + *err);
  horizon = h;
}

void Runtime::alloc_worker(Gpu& G, int id) {
  G.id = id;
  G.dev = id % ndev;
  set_dev(G);
  int lo = 0, hi = 0;
  RP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));  // lo = least, hi = greatest
  auto mk = [&](cudaStream_t* st, int prio) {
    RP_CUDA(cudaStreamCreateWithPriority(st, cudaStreamNonBlocking, prio));
  };
  mk(&G.compute, hi);
  mk(&G.act, hi);
  mk(&G.wgrad, hi + 1 <= lo ? hi + 1 : hi);
  mk(&G.w_h2d, lo);
  mk(&G.opt_h2d, lo);
  mk(&G.opt_d2h, lo);
  mk(&G.opt_comp, lo);
  mk(&G.opt_res, lo);
  G.allocated.assign(8, 0);
  auto dalloc = [&](std::size_t bytes, int cat) -> void* { return this->dalloc(G, bytes, cat); };
  const int64_t Th = (int64_t)T * s.h;
  const int64_t Tk = (int64_t)T * (s.moe() ? s.ek : 1);  // rows of the (expert-sorted) MLP buffers
  G.groups.resize(ngroups());
  for (int g = 0; g < ngroups(); ++g) {
    DevGroup& D = G.groups[g];
    const int64_t n = group_numel(g);
    for (int b = 0; b < 2; ++b) {
      if (!pooled) D.w[b] = static_cast<uint16_t*>(dalloc(n * 2, 0));
      D.ev_upload[b] = new_event(false);
      D.ev_lastuse[b] = new_event(false);
    }
    const int64_t tn = host[g].tn(), to = host[g].t_off;  // trainable region only
    if (!pooled) {
      D.grad[0] = tn > 0 ? static_cast<float*>(dalloc(tn * 4, 1)) - to : nullptr;
      D.grad[1] = tn > 0 ? static_cast<float*>(dalloc(tn * 4, 1)) - to : nullptr;
      // AdamW output: the trainable region only (indexed from t_off like grads)
      D.pend = static_cast<uint16_t*>(dalloc(tn * 2, 2)) - to;
    }
    D.ev_gradwrite = new_event(false);
    D.ev_adam[0] = new_event(false);
    D.ev_adam[1] = new_event(false);
    D.ev_pcopy = new_event(false);
  }
  const int nsets = std::max(1, s.L - plan.fused_stage.first);
  G.acts.resize(nsets);
  // opt-in (RP_FUSED_PIPELINE=1): measured no faster at Qwen3-8B, where the
  // step runs at the 1 kW power cap (the overlap lowers SM clocks instead),
  // while the second activation set costs 20.6 GB of HBM that otherwise holds
  // optimizer state
  const bool pipe = plan.fused_stage.first == 0 && MR >= 2 && !s.moe() &&
                    (cfg.flags & RP_RT_FUSED_PIPELINE);  // (MoE scratch is single-stream)
  if (pipe) G.acts2.resize(nsets);
  for (auto* set : {&G.acts, &G.acts2})
  for (auto& A : *set) {
    A.x = static_cast<uint16_t*>(dalloc(Th * 2, 3));
    A.h1 = static_cast<uint16_t*>(dalloc(Th * 2, 3));
    A.qkv = static_cast<uint16_t*>(dalloc((int64_t)T * s.qkvd() * 2, 3));
    A.q = static_cast<uint16_t*>(dalloc((int64_t)T * s.qd() * 2, 3));
    A.k = static_cast<uint16_t*>(dalloc((int64_t)T * s.kd() * 2, 3));
    A.o = static_cast<uint16_t*>(dalloc((int64_t)T * s.qd() * 2, 3));
    A.x2 = static_cast<uint16_t*>(dalloc(Th * 2, 3));
    A.h2 = static_cast<uint16_t*>(dalloc(Th * 2, 3));
    A.gu = static_cast<uint16_t*>(dalloc(Tk * 2 * s.m * 2, 3));
    A.act = static_cast<uint16_t*>(dalloc(Tk * s.m * 2, 3));
    A.rstd1 = static_cast<float*>(dalloc((std::size_t)T * 4, 3));
    A.rstd2 = static_cast<float*>(dalloc((std::size_t)T * 4, 3));
    A.rstd_q = static_cast<float*>(dalloc((int64_t)T * s.nq * 4, 3));
    A.rstd_k = static_cast<float*>(dalloc((int64_t)T * s.nk * 4, 3));
    A.lse = static_cast<float*>(dalloc((int64_t)T * s.nq * 4, 3));
    A.ev_free = new_event(false);
    A.ev_chain_free = new_event(false);
    if (lora_r) {
      A.u_qkv = static_cast<uint16_t*>(dalloc((int64_t)T * lora_r * 2, 3));
      A.u_o = static_cast<uint16_t*>(dalloc((int64_t)T * lora_r * 2, 3));
      if (!s.moe()) {
        A.u_gu = static_cast<uint16_t*>(dalloc((int64_t)T * lora_r * 2, 3));
        A.u_down = static_cast<uint16_t*>(dalloc((int64_t)T * lora_r * 2, 3));
      }
    }
    if (s.moe()) {
      A.r_logits = static_cast<float*>(dalloc((int64_t)T * s.E * 4, 3));
      A.r_idx = static_cast<int32_t*>(dalloc((int64_t)T * s.ek * 4, 3));
      A.r_w = static_cast<float*>(dalloc((int64_t)T * s.ek * 4, 3));
      A.r_pos = static_cast<int32_t*>(dalloc((int64_t)T * s.ek * 4, 3));
      A.r_ws = static_cast<float*>(dalloc(Tk * 4, 3));
      A.r_off = static_cast<int32_t*>(dalloc((int64_t)(s.E + 1) * 4, 3));
    }
  }
  if (s.moe()) {
    G.m_xs = static_cast<uint16_t*>(dalloc(Tk * s.h * 2, 4));
    G.m_ys = static_cast<uint16_t*>(dalloc(Tk * s.h * 2, 4));
    G.m_dact = static_cast<uint16_t*>(dalloc(Tk * s.m * 2, 4));
    G.m_dlogits = static_cast<uint16_t*>(dalloc((int64_t)T * s.E * 2, 4));
    G.m_counts = static_cast<int32_t*>(dalloc((int64_t)s.E * 4, 4));
    G.m_cursor = static_cast<int32_t*>(dalloc((int64_t)s.E * 4, 4));
    G.m_dws = static_cast<float*>(dalloc(Tk * 4, 4));
    G.m_dh32 = static_cast<float*>(dalloc(Th * 4, 4));
  }
  if (lora_r) G.du = static_cast<uint16_t*>(dalloc((int64_t)T * lora_r * 2, 4));
  if (pipe) {
    int lo2 = 0, hi2 = 0;
    RP_CUDA(cudaDeviceGetStreamPriorityRange(&lo2, &hi2));
    RP_CUDA(cudaStreamCreateWithPriority(&G.fwd2, cudaStreamNonBlocking, hi2));
    G.hdx32 = static_cast<float*>(dalloc(Th * 4, 4));
    G.hdx16 = static_cast<uint16_t*>(dalloc(Th * 2, 4));
    G.hdh = static_cast<uint16_t*>(dalloc(Th * 2, 4));
    G.ev_head_done = new_event(false);
    G.ev_hdx_free = new_event(false);
    G.ev_fwd_join = new_event(false);
  }
  G.dx32[0] = static_cast<float*>(dalloc(Th * 4, 4));
  G.dx32[1] = static_cast<float*>(dalloc(Th * 4, 4));
  for (int b = 0; b < 2; ++b) {
    G.dx16s[b] = static_cast<uint16_t*>(dalloc(Th * 2, 4));
    G.dqkvs[b] = static_cast<uint16_t*>(dalloc((int64_t)T * s.qkvd() * 2, 4));
    G.ev_dx16_free[b] = new_event(false);
    G.ev_dqkv_free[b] = new_event(false);
  }
  for (int b = 0; b < G.n_dgu; ++b) {
    G.dgus[b] = static_cast<uint16_t*>(dalloc(Tk * 2 * s.m * 2, 4));
    G.ev_dgu_free[b] = new_event(false);
  }
  G.ev_wgrad = new_event(false);
  G.dx16 = G.dx16s[0];
  G.dh = static_cast<uint16_t*>(dalloc(Th * 2, 4));
  G.dact = static_cast<uint16_t*>(dalloc((int64_t)T * s.m * 2, 4));
  G.dattn = static_cast<uint16_t*>(dalloc((int64_t)T * s.qd() * 2, 4));
  G.dq_t = static_cast<uint16_t*>(dalloc((int64_t)T * s.qd() * 2, 4));
  G.dk_t = static_cast<uint16_t*>(dalloc((int64_t)T * s.kd() * 2, 4));
  G.dq_acc = static_cast<float*>(dalloc((int64_t)T * s.qd() * 4, 4));
  G.delta = static_cast<float*>(dalloc((int64_t)T * s.nq * 4, 4));
  G.xbuf[0] = static_cast<uint16_t*>(dalloc(Th * 2, 4));
  G.xbuf[1] = static_cast<uint16_t*>(dalloc(Th * 2, 4));
  G.hN = static_cast<uint16_t*>(dalloc(Th * 2, 4));
  G.rstdN = static_cast<float*>(dalloc((std::size_t)T * 4, 4));
  G.logits = static_cast<uint16_t*>(dalloc((int64_t)std::min(T, logits_rows) * s.V * 2, 4));
  for (int b = 0; b < 2; ++b) {
    G.loss_par[b] = static_cast<float*>(dalloc(64, 4));
    G.tokens_par[b] = static_cast<int32_t*>(dalloc((int64_t)M * T * 4, 4));
    G.labels_par[b] = static_cast<int32_t*>(dalloc((int64_t)M * T * 4, 4));
    G.ev_iter_done[b] = new_event(false);
    G.ev_loss_par[b] = new_event(false);
  }
  G.loss_dev = G.loss_par[0];
  G.tokens_dev = G.tokens_par[0];
  G.labels_dev = G.labels_par[0];
  G.ev_tokens = new_event(false);
  {  // RoPE (cos, sin) table: float64 on the host, rounded (as the oracle)
    const int half = s.hd / 2;
    std::vector<float> tab((std::size_t)cfg.seq_len * half * 2);
    for (int p = 0; p < cfg.seq_len; ++p)
      for (int j = 0; j < half; ++j) {
        const double inv = 1.0 / std::pow(s.theta, (2.0 * j) / s.hd);
        tab[((std::size_t)p * half + j) * 2] = (float)std::cos(p * inv);
        tab[((std::size_t)p * half + j) * 2 + 1] = (float)std::sin(p * inv);
      }
    G.cos_sin = static_cast<float*>(dalloc(tab.size() * 4, 4));
    RP_CUDA(cudaMemcpy(G.cos_sin, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
  }
  if (S > 1) {  // hand-off and checkpoint buffers
    auto mkbuf = [&](std::size_t bytes, int cat) {  // cat < 0: pooled (bound on demand)
      Slotbuf b;
      b.p = cat < 0 ? nullptr : dalloc(bytes, cat);
      b.ready_dev.assign(ndev, nullptr);
      b.read = new_event(false);
      return b;
    };
    for (int p = 0; p < parities; ++p)
      for (int mb = 0; mb < MR; ++mb) {
        G.hand_act.push_back(mkbuf(Th * 2, 5));
        G.hand_grad.push_back(mkbuf(Th * 4, 5));
      }
    G.ckpt.resize((std::size_t)parities * s.L * MR);
    for (int p = 0; p < parities; ++p)
      for (int l = 0; l < plan.fused_stage.first && l < s.L; ++l)
        for (int mb = 0; mb < MR; ++mb)
          G.ckpt[((std::size_t)p * s.L + l) * MR + mb] = mkbuf(Th * 2, pooled ? -1 : 5);
  }
  for (int b = 0; b < Gpu::kOptSlots; ++b) {
    for (int j = 0; j < 3; ++j)
      G.opt_buf[b][j] = static_cast<float*>(dalloc((std::size_t)chunk_elems * 4, 6));
    G.opt_free[b] = new_event(false);
  }
  G.anchor = new_event(true);
  RP_CUDA(cudaEventRecord(G.anchor, G.compute));
}

// ---- weight init (bench path; tests load weights through rp_set_params) ----------
void Runtime::init_weights() {
  Gpu& G = gpus[0];
  set_dev(G);
  const float std_ = cfg.init_std > 0 ? cfg.init_std : 0.02f;
  int64_t nmax = 0;
  for (int g = 0; g < ngroups(); ++g) nmax = std::max(nmax, host[g].n);
  float* f32 = nullptr;  // fp32 + bf16 scratch of the largest group
  uint16_t* b16 = nullptr;
  RP_CUDA(cudaMalloc(&f32, (std::size_t)nmax * 4));
  RP_CUDA(cudaMalloc(&b16, (std::size_t)nmax * 2));
  for (int g = 0; g < ngroups(); ++g) {
    HostGroup& H = host[g];
    RP_K(rp_init_normal(f32, b16, H.n, cfg.init_seed * 1000003ull + (uint64_t)g, std_,
                        G.compute));
    std::vector<std::pair<int64_t, int64_t>> ones, zeros;
    if (g >= 1 && g <= s.L) {
      ones = {{LL.in_norm.off, s.h}, {LL.q_norm.off, s.hd}, {LL.k_norm.off, s.hd},
              {LL.post_norm.off, s.h}};
      if (lora_r)  // LoRA B starts at zero (the adapted model starts as the base)
        for (const Tensor* t : {&LL.qkv_B, &LL.o_B, &LL.gu_B, &LL.down_B})
          if (t->numel() > 0) zeros.emplace_back(t->off, t->numel());
    } else if (g == s.L + 1) {
      ones = {{HL.final_norm.off, s.h}};
    }
    for (auto [off, n] : ones) RP_K(rp_fill(f32 + off, b16 + off, n, 1.0f, G.compute));
    for (auto [off, n] : zeros) RP_K(rp_fill(f32 + off, b16 + off, n, 0.0f, G.compute));
    if (H.tn() > 0)
      RP_CUDA(cudaMemcpyAsync(H.master + H.t_off, f32 + H.t_off, H.tn() * 4,
                              cudaMemcpyDeviceToHost, G.compute));
    RP_CUDA(cudaMemcpyAsync(H.w16, b16, H.n * 2, cudaMemcpyDeviceToHost, G.compute));
    RP_CUDA(cudaStreamSynchronize(G.compute));
  }
  RP_CUDA(cudaFree(f32));
  RP_CUDA(cudaFree(b16));
}

// ---- GPU lane: weight upload ----------------------------------------------------------
// upload(l, t): bf16 master (pinned host) -> worker weights, on the
// low-priority H2D stream, after p_copy(l, t-1) (edge 2) and after the last
// compute read of the previous version (WAR). A worker that already holds
// this iteration's version skips the copy. After the LAST upload of the
// group in the iteration, the pending AdamW result may be published
// (p_copy, edge 1) — async mode only.
void Runtime::upload(Gpu& G, int g, int it, bool last_use) {
  if (upload_reserve(G, g, it)) {
    upload_chunk(G, g, it, 0, host[g].n * 2);
    upload_done(G, g, it);
  }
  if (last_use && cfg.async_optimizer && pend_owner[g] >= 0) p_copy(g);
  set_dev(G);
}

// The upload of (g, it) into w[it%2] of worker G is now the runtime's job:
// returns true when a host copy is needed (the caller then enqueues its
// chunks and upload_done); false when the worker already holds version it.
bool Runtime::upload_reserve(Gpu& G, int g, int it) {
  DevGroup& D = G.groups[g];
  HostGroup& H = host[g];
  const int b = it & 1;
  if (D.loaded[b] != it && H.direct && H.w16_stale) {
    // direct group without a new update for `it` (no step() in between): the
    // latest version lives in the other device buffer
    set_dev(G);
    RP_CUDA(cudaStreamWaitEvent(G.w_h2d, D.ev_lastuse[b], 0));
    RP_CUDA(cudaStreamWaitEvent(G.w_h2d, D.ev_upload[b ^ 1], 0));
    RP_CUDA(cudaMemcpyAsync(D.w[b], D.w[b ^ 1], H.n * 2, cudaMemcpyDeviceToDevice, G.w_h2d));
    RP_CUDA(cudaEventRecord(D.ev_upload[b], G.w_h2d));
    D.loaded[b] = it;
  }
  upload_ver[g] = std::max(upload_ver[g], it);
  if (D.loaded[b] == it) return false;
  if (pooled && !D.w[b]) {  // a slab of the worker's pool for this version
    D.w_slab[b] = slab_acquire(G, (std::size_t)H.n * 2, 0, G.w_h2d);
    D.w[b] = static_cast<uint16_t*>(G.slabs[D.w_slab[b]].p);
  }
  D.loaded[b] = it;  // reserved: the chunks follow (possibly window by window)
  D.up_started = false;
  return true;
}

// One chunk [off, off+len) bytes of group g's bf16 weights, pinned host
// master -> worker G, on the low-priority H2D stream. The first chunk of an
// upload carries its waits: edge (2) — the group's published-version flag
// word — and the WAR wait on the buffer's previous version.
void Runtime::upload_chunk(Gpu& G, int g, int it, int64_t off, int64_t len) {
  DevGroup& D = G.groups[g];
  HostGroup& H = host[g];
  const int b = it & 1;
  set_dev(G);
  if (!D.up_started) {
    if (pcopy_idx[g] >= 0) {  // edge (2): the host master holds the published version
      flags.wait_geq(G.w_h2d, flag_pub(g), (uint32_t)pcopy_idx[g] + 1);
      proto_edge(roundpipe::ActionKind::ParamCopy, g, pcopy_idx[g],
                 roundpipe::ActionKind::ParamUpload, g, it);
    }
    RP_CUDA(cudaStreamWaitEvent(G.w_h2d, D.ev_lastuse[b], 0));  // WAR (t-2)
    D.up_xa = xfer_begin(G.w_h2d);
    D.up_started = true;
  }
  RP_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(D.w[b]) + off,
                          reinterpret_cast<const uint8_t*>(H.w16) + off, (std::size_t)len,
                          cudaMemcpyHostToDevice, G.w_h2d));
  h2d_bytes += len;
}

void Runtime::upload_done(Gpu& G, int g, int it) {
  DevGroup& D = G.groups[g];
  const int b = it & 1;
  set_dev(G);
  xfer_end(D.up_xa, G.w_h2d, 0, g - 1, it, G.id);
  RP_CUDA(cudaEventRecord(D.ev_upload[b], G.w_h2d));
  uploaders[g].push_back(G.id * 2 + b);
}

// LPT transfer windows: the uploads of iteration it+1 are
// cut with the reference transfer planner (transfer_planner::plan: tensors
// sorted by size, chunked to ceil(total/W), each chunk to the least-loaded
// window) into one window per micro-batch task worker G runs in iteration
// it; window k is released onto the low-priority H2D stream when G's compute
// starts its k-th micro-batch, so parameter traffic is paced by compute and
// spread over the iteration instead of queued in one burst. A worker without
// tasks in iteration it gets everything at once.
void Runtime::plan_upload_windows(int it_next) {
  ensure_horizon(it_next);
  std::vector<std::vector<int>> todo(N);  // per worker, groups in use order
  std::vector<int> wins(N, 0);
  for (std::size_t i = 0; i < sched.tasks.size();) {
    const roundpipe::Task& t = sched.tasks[i];
    if (t.iteration > it_next) break;
    if (t.iteration == it_next - 1) wins[t.gpu] += MR;
    if (t.iteration == it_next)
      for (int g : slot_groups(slots[t.slot])) todo[t.gpu].push_back(g);
    i += MR;
  }
  for (int w = 0; w < N; ++w) {
    Gpu& G = gpus[w];
    std::vector<roundpipe::TransferItem> items;
    std::vector<std::pair<int, int64_t>> tensor;  // item -> (group, byte offset)
    for (int g : todo[w]) {
      if (!upload_reserve(G, g, it_next)) continue;
      // the group's tensors (weights of one layer / the head / the table)
      std::vector<Tensor> ts;
      if (g == 0) ts = {Tensor{0, s.V, s.h}};
      else if (g == s.L + 1) ts = {HL.final_norm, HL.lm_head};
      else ts = {LL.in_norm, LL.qkv, LL.q_norm, LL.k_norm, LL.o, LL.post_norm, LL.gate_up, LL.down};
      const int64_t end = host[g].n * 2;
      for (std::size_t k = 0; k < ts.size(); ++k) {  // tensor k spans to the next tensor's offset
        const int64_t a = ts[k].off * 2;
        const int64_t z = k + 1 < ts.size() ? ts[k + 1].off * 2 : end;
        items.push_back({"g" + std::to_string(g) + "." + std::to_string(k), z - a,
                         roundpipe::TransferDirection::Upload, 0});
        tensor.push_back({g, a});
      }
    }
    if (items.empty()) continue;
    std::unordered_map<std::string, std::size_t> idx;
    for (std::size_t k = 0; k < items.size(); ++k) idx[items[k].tensor_id] = k;
    auto& left = up_left[w];
    if (wins[w] == 0) {  // no compute to pace against: all now
      for (std::size_t k = 0; k < items.size(); ++k) ++left[tensor[k].first];
      for (std::size_t k = 0; k < items.size(); ++k) {
        const int g = tensor[k].first;
        upload_chunk(G, g, it_next, tensor[k].second, items[k].bytes);
        if (--left[g] == 0) upload_done(G, g, it_next);
      }
      continue;
    }
    const int64_t max_chunk = roundpipe::transfer_planner::default_max_chunk(items, wins[w]);
    const auto plan = roundpipe::transfer_planner::plan(items, wins[w], max_chunk);
    for (const auto& win : plan.windows) {
      UpWindow uw;
      uw.it = it_next;
      for (const auto& c : win.items) {
        const auto [g, base] = tensor[idx.at(c.tensor_id)];
        uw.chunks.push_back({g, base + (int64_t)c.chunk_index * max_chunk, c.bytes});
        ++left[g];
      }
      upq[w].push_back(std::move(uw));
    }
  }
}

// Worker G's compute is about to start a micro-batch: release the next
// upload window onto the H2D stream behind that point of the compute stream.
void Runtime::release_window(Gpu& G) {
  if (upq[G.id].empty()) return;
  UpWindow uw = std::move(upq[G.id].front());
  upq[G.id].pop_front();
  if (!uw.chunks.empty()) join(G, G.compute, G.w_h2d);
  auto& left = up_left[G.id];
  for (const auto& c : uw.chunks) {
    upload_chunk(G, c.g, uw.it, c.off, c.len);
    if (--left[c.g] == 0) upload_done(G, c.g, uw.it);
  }
}

void Runtime::flush_windows() {
  for (Gpu& G : gpus)
    while (!upq[G.id].empty()) release_window(G);
}

// Enqueue iteration it's weight uploads ahead of time (into the other
// parity buffer) so they stream in under the current iteration's compute.
void Runtime::prefetch(int it, bool reverse) {
  ensure_horizon(it);
  std::vector<std::pair<int, int>> todo;  // (worker, group) in use order
  for (std::size_t i = 0; i < sched.tasks.size();) {
    const roundpipe::Task& t = sched.tasks[i];
    if (t.iteration < it) { ++i; continue; }
    if (t.iteration > it) break;
    for (int g : slot_groups(slots[t.slot])) todo.emplace_back(t.gpu, g);
    i += MR;
  }
  if (reverse) std::reverse(todo.begin(), todo.end());
  for (auto [w, g] : todo) upload(gpus[w], g, it, false);
}

// Parameter groups a slot reads, in the order its compute needs them.
std::vector<int> Runtime::slot_groups(const roundpipe::StageSlot& ss) const {
  std::vector<int> gs;
  const int a = ss.layers.first, b = ss.layers.last;
  if (ss.kind != StageKind::Backward && a == 0) gs.push_back(0);
  if (ss.kind == StageKind::Backward)
    for (int l = b; l >= a; --l) gs.push_back(l + 1);
  else
    for (int l = a; l <= b; ++l) gs.push_back(l + 1);
  return gs;
}

// p_copy: pending AdamW result (device) -> bf16 master (pinned host), after
// every upload of the current version (edge 1).
void Runtime::p_copy(int g) {
  Gpu& O = gpus[pend_owner[g]];
  set_dev(O);
  DevGroup& D = O.groups[g];
  HostGroup& H = host[g];
  // ParamCopy index = the version whose uploads this publication follows
  const int idx = upload_ver[g];
  for (int wb : uploaders[g])  // edge (1)
    RP_CUDA(cudaStreamWaitEvent(O.opt_d2h, gpus[wb / 2].groups[g].ev_upload[wb % 2], 0));
  if (!uploaders[g].empty())
    proto_edge(roundpipe::ActionKind::ParamUpload, g, idx, roundpipe::ActionKind::ParamCopy, g,
               idx);
  uploaders[g].clear();
  RP_CUDA(cudaStreamWaitEvent(O.opt_d2h, D.ev_adam[0], 0));
  RP_CUDA(cudaStreamWaitEvent(O.opt_d2h, D.ev_adam[1], 0));
  cudaEvent_t xa = xfer_begin(O.opt_d2h);
  RP_CUDA(cudaMemcpyAsync(H.w16 + H.t_off, D.pend + H.t_off, H.tn() * 2, cudaMemcpyDeviceToHost,
                          O.opt_d2h));  // frozen parts never change
  xfer_end(xa, O.opt_d2h, 1, g - 1, H.step, O.id);
  d2h_bytes += H.tn() * 2;
  RP_CUDA(cudaEventRecord(D.ev_pcopy, O.opt_d2h));
  flags.set(O.opt_d2h, flag_pub(g), (uint32_t)idx + 1);
  if (pooled && D.pend_slab >= 0) {
    slab_release(O, D.pend_slab, O.opt_d2h);
    D.pend_slab = -1;
    D.pend = nullptr;
  }
  pcopy_idx[g] = idx;
  pend_owner[g] = -1;
}

// ---- decoder layer -------------------------------------------------------------------
void Runtime::layer_fwd(Gpu& G, int l, const uint16_t* x, LayerActs& A, uint16_t* x_out,
                        cudaStream_t on) {
  const uint16_t* W = G.groups[l + 1].w[exec_iter & 1];
  cudaStream_t st = on ? on : G.compute;
  const int h = s.h, qd = s.qd(), kd = s.kd(), qkvd = s.qkvd();
  RP_CUDA(cudaStreamWaitEvent(st, A.ev_free, 0));        // last weight-gradient reads of A
  RP_CUDA(cudaStreamWaitEvent(st, A.ev_chain_free, 0));  // last dgrad-chain reads of A
  A.xin = x;
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_rmsnorm_fwd(x, h, W + LL.in_norm.off, A.h1, h, A.rstd1, T, h, (float)s.eps, st));
    prof_end(pi_, st, 2, 4.0 * T * h);
  }
  lin_fwd(st, W, LL.qkv, &LL.qkv_A, &LL.qkv_B, A.h1, h, h, A.u_qkv, A.qkv, qkvd, qkvd);
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_qk_norm_rope_fwd(A.qkv, qkvd, s.nq, s.nk, s.hd, W + LL.q_norm.off, W + LL.k_norm.off,
                           G.cos_sin, cfg.seq_len, A.q, A.k, A.rstd_q, A.rstd_k, T, (float)s.eps,
                           st));
    prof_end(pi_, st, 2, 4.0 * T * (s.nq + s.nk) * s.hd);
  }
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_attn_fwd_tc(A.q, qd, A.k, kd, A.qkv + qd + kd, qkvd, A.o, qd, A.lse, T, cfg.seq_len, s.nq,
                   s.nk, s.hd, 1.0f / std::sqrt((float)s.hd), st));
    prof_end(pi_, st, 1, 2.0 * s.nq * s.hd * (double)T * cfg.seq_len);
  }
  lin_fwd(st, W, LL.o, &LL.o_A, &LL.o_B, A.o, qd, qd, A.u_o, A.x2, h, h, x, h);
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_rmsnorm_fwd(A.x2, h, W + LL.post_norm.off, A.h2, h, A.rstd2, T, h, (float)s.eps, st));
    prof_end(pi_, st, 2, 4.0 * T * h);
  }
  if (s.moe()) {  // routed experts instead of the dense MLP
    moe_mlp_fwd(G, st, W, A, x_out);
    kernels += 5;
    return;
  }
  const bool unfused = cfg.flags & RP_RT_UNFUSED_SWIGLU;
  if (lora_r && !unfused && T >= 256) {  // LoRA: Us first, then the dual GEMM with [X | Us]
    const int r = lora_r;
    gemm(st, A.h2, h, false, W + LL.gu_A.off, h, false, A.u_gu, r, false, false, T, r, h);
    RP_K(rp_scale_bf16(A.u_gu, (int64_t)T * r, lora_scale, st));
    rp_gemm_args_t a{};
    a.M = T;
    a.N = s.m;
    a.K = h;
    a.A = A.h2;
    a.lda = h;
    a.B = W + LL.gate_up.off;
    a.ldb = h;
    a.D = A.gu;
    a.ldd = 2 * s.m;
    const int pi_ = prof_begin(st);
    RP_K(rp_gemm_ex(&a, 2, A.act, s.m, A.u_gu, r, W + LL.gu_B.off, r, r, st));
    prof_end(pi_, st, 0, 2.0 * T * 2 * s.m * (double)(h + r));
    kernels += 2;
  } else if (!lora_r && !unfused) {  // SwiGLU in the gate/up GEMM's epilogue (gu kept for bwd)
    rp_gemm_args_t a{};
    a.M = T;
    a.N = s.m;
    a.K = h;
    a.A = A.h2;
    a.lda = h;
    a.B = W + LL.gate_up.off;
    a.ldb = h;
    a.D = A.gu;
    a.ldd = 2 * s.m;
    const int pi_ = prof_begin(st);
    RP_K(rp_gemm_swiglu_fwd(&a, A.act, s.m, st));
    prof_end(pi_, st, 0, 2.0 * T * 2 * s.m * (double)h);
    ++kernels;
  } else {
    lin_fwd(st, W, LL.gate_up, &LL.gu_A, &LL.gu_B, A.h2, h, h, A.u_gu, A.gu, 2 * s.m, 2 * s.m);
    const int pi_ = prof_begin(st);
    RP_K(rp_swiglu_fwd(A.gu, A.act, T, s.m, st));
    prof_end(pi_, st, 2, 6.0 * T * s.m);
  }
  lin_fwd(st, W, LL.down, &LL.down_A, &LL.down_B, A.act, s.m, s.m, A.u_down, x_out, h, h, A.x2,
          h);
  kernels += 5;
}

// Backward of decoder layer l. In: G.dx32[0] (fp32) / G.dx16 (bf16) =
// dL/d(layer output). Out: the same buffers = dL/d(layer input). Weight grads
// go to grad[t%2]: the first micro-batch overwrites, later ones accumulate.
// The dgrad chain runs on `compute`; the four weight-gradient GEMMs run on the
// `wgrad` stream as soon as their inputs exist (event per input), so they fill
// the persistent GEMMs' partial last waves and overlap the chain's
// elementwise / attention kernels. Buffers they read are double-buffered
// (dx16 A/B, dgu and dqkv by layer parity) and released by events.
void Runtime::layer_bwd(Gpu& G, int l, LayerActs& A, bool first) {
  DevGroup& D = G.groups[l + 1];
  const uint16_t* W = D.w[exec_iter & 1];
  float* dW = D.grad[last_iter & 1];
  // profiled steps serialise the weight-gradient GEMMs onto `compute` so each
  // kernel's CUDA-event time is its own (the timed steps overlap them)
  cudaStream_t st = G.compute, ws = prof_on ? G.compute : G.wgrad;
  const int h = s.h, m = s.m, qd = s.qd(), kd = s.kd(), qkvd = s.qkvd();
  const int xa = G.dx16 == G.dx16s[0] ? 0 : 1, xb = xa ^ 1;  // dY in, post-norm dY
  uint16_t* dx_a = G.dx16s[xa];
  uint16_t* dx_b = G.dx16s[xb];
  const int p = G.bwd_par;
  G.bwd_par ^= 1;
  const int pg = G.dgu_i;
  G.dgu_i = (G.dgu_i + 1) % G.n_dgu;
  uint16_t* dgu = G.dgus[pg];
  uint16_t* dqkv = G.dqkvs[p];
  auto to_ws = [&]() { join(G, st, ws); };  // wgrad waits for everything on compute so far
  const bool full = lora_r == 0;  // LoRA: base weights frozen, adapters trained
  if (first) {
    grad_free(G, l + 1, st);
    if (full)
      for (const Tensor* t : {&LL.in_norm, &LL.q_norm, &LL.k_norm, &LL.post_norm})
        RP_CUDA(cudaMemsetAsync(dW + t->off, 0, t->numel() * 4, st));
  }
  // MLP:  x3 = x2 + act(gu(h2)) Wd^T
  if (s.moe()) {  // routed experts (frozen): dh = d(h2) through experts and router
    RP_CUDA(cudaStreamWaitEvent(st, G.ev_dgu_free[pg], 0));
    moe_mlp_bwd(G, st, W, A, dx_a, dgu);
    RP_CUDA(cudaEventRecord(G.ev_dx16_free[xa], st));
    RP_CUDA(cudaEventRecord(G.ev_dgu_free[pg], st));
  } else {
  to_ws();
  if (full) gemm(ws, dx_a, h, true, A.act, m, true, dW + LL.down.off, m, true, !first, h, m, T);
  // full fine-tune: the SwiGLU backward runs in the dgrad GEMM's epilogue
  // (dact never reaches HBM); LoRA adds the adapter term to dact first
  const bool unfused = cfg.flags & RP_RT_UNFUSED_SWIGLU;
  const bool fuse = full && !unfused;
  const bool lora_fuse = !full && !unfused && T >= 256;
  RP_CUDA(cudaStreamWaitEvent(st, G.ev_dgu_free[pg], 0));  // wgrad n_dgu layers ago read it
  if (fuse) {
    gemm(st, dx_a, h, false, W + LL.down.off, m, true, dgu, 2 * m, false, false, T, m, h, A.gu,
         2 * m, true);
  } else if (full) {
    gemm(st, dx_a, h, false, W + LL.down.off, m, true, G.dact, m, false, false, T, m, h);
  } else if (lora_fuse) {  // dUs = s dY B, then dgu from [dY | dUs] [Wd ; A] in one GEMM
    const int r = lora_r;
    gemm(st, dx_a, h, false, W + LL.down_B.off, r, true, G.du, r, false, false, T, r, h);
    RP_K(rp_scale_bf16(G.du, (int64_t)T * r, lora_scale, st));
    rp_gemm_args_t a{};
    a.M = T;
    a.N = m;
    a.K = h;
    a.A = dx_a;
    a.lda = h;
    a.B = W + LL.down.off;
    a.ldb = m;
    a.b_mn_major = 1;
    a.D = dgu;
    a.ldd = 2 * m;
    a.R = A.gu;
    a.ldr = 2 * m;
    const int pi_ = prof_begin(st);
    RP_K(rp_gemm_ex(&a, 1, nullptr, 0, G.du, r, W + LL.down_A.off, m, r, st));
    prof_end(pi_, st, 0, 2.0 * T * m * (double)(h + r));
    kernels += 2;
    lora_wgrad(G, st, dW, LL.down_A, LL.down_B, A.act, m, m, A.u_down, dx_a, h, h, first);
  } else {
    lin_dgrad(G, st, W, LL.down, &LL.down_A, &LL.down_B, dx_a, h, h, G.dact, m, m);
    lora_wgrad(G, st, dW, LL.down_A, LL.down_B, A.act, m, m, A.u_down, dx_a, h, h, first);
  }
  RP_CUDA(cudaEventRecord(G.ev_dx16_free[xa], full ? ws : st));
  if (!fuse && !lora_fuse) {
    const int pi_ = prof_begin(st);
    RP_K(rp_swiglu_bwd(G.dact, A.gu, dgu, T, m, st));
    prof_end(pi_, st, 2, 10.0 * T * m);
  }
  to_ws();
  if (full)
    gemm(ws, dgu, 2 * m, true, A.h2, h, true, dW + LL.gate_up.off, h, true, !first, 2 * m, h, T);
  RP_CUDA(cudaEventRecord(G.ev_dgu_free[pg], full ? ws : st));
  if (full) {
    gemm(st, dgu, 2 * m, false, W + LL.gate_up.off, h, true, G.dh, h, false, false, T, h, 2 * m);
  } else {
    lin_dgrad(G, st, W, LL.gate_up, &LL.gu_A, &LL.gu_B, dgu, 2 * m, 2 * m, G.dh, h, h);
    lora_wgrad(G, st, dW, LL.gu_A, LL.gu_B, A.h2, h, h, A.u_gu, dgu, 2 * m, 2 * m, first);
  }
  }  // dense MLP
  RP_CUDA(cudaStreamWaitEvent(st, G.ev_dx16_free[xb], 0));
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_rmsnorm_bwd(G.dh, A.x2, W + LL.post_norm.off, A.rstd2, G.dx32[0], G.dx32[1], dx_b,
                        full ? dW + LL.post_norm.off : nullptr, T, h, st));
    prof_end(pi_, st, 2, 14.0 * T * h);
  }
  // attention:  x2 = x + attn(qkv(h1)) Wo^T
  to_ws();
  if (full) gemm(ws, dx_b, h, true, A.o, qd, true, dW + LL.o.off, qd, true, !first, h, qd, T);
  if (full) {
    gemm(st, dx_b, h, false, W + LL.o.off, qd, true, G.dattn, qd, false, false, T, qd, h);
  } else {
    lin_dgrad(G, st, W, LL.o, &LL.o_A, &LL.o_B, dx_b, h, h, G.dattn, qd, qd);
    lora_wgrad(G, st, dW, LL.o_A, LL.o_B, A.o, qd, qd, A.u_o, dx_b, h, h, first);
  }
  RP_CUDA(cudaEventRecord(G.ev_dx16_free[xb], full ? ws : st));
  RP_CUDA(cudaStreamWaitEvent(st, G.ev_dqkv_free[p], 0));
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_attn_bwd_tc(A.q, qd, A.k, kd, A.qkv + qd + kd, qkvd, A.o, qd, G.dattn, qd, A.lse,
                        G.dq_t, qd, G.dk_t, kd, dqkv + qd + kd, qkvd, G.delta, G.dq_acc, T,
                        cfg.seq_len, s.nq, s.nk, s.hd, 1.0f / std::sqrt((float)s.hd), st));
    prof_end(pi_, st, 1, 5.0 * s.nq * s.hd * (double)T * cfg.seq_len);
  }
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_qk_norm_rope_bwd(G.dq_t, G.dk_t, A.qkv, qkvd, s.nq, s.nk, s.hd, W + LL.q_norm.off,
                             W + LL.k_norm.off, A.rstd_q, A.rstd_k, G.cos_sin, cfg.seq_len, dqkv,
                             qkvd, full ? dW + LL.q_norm.off : nullptr,
                             full ? dW + LL.k_norm.off : nullptr, T, st));
    prof_end(pi_, st, 2, 8.0 * T * (s.nq + s.nk) * s.hd);
  }
  to_ws();
  if (full)
    gemm(ws, dqkv, qkvd, true, A.h1, h, true, dW + LL.qkv.off, h, true, !first, qkvd, h, T);
  RP_CUDA(cudaEventRecord(G.ev_dqkv_free[p], ws));
  RP_CUDA(cudaEventRecord(A.ev_free, ws));  // act / h2 / o / h1 no longer needed
  RP_CUDA(cudaEventRecord(G.ev_wgrad, ws));
  if (full) {
    gemm(st, dqkv, qkvd, false, W + LL.qkv.off, h, true, G.dh, h, false, false, T, h, qkvd);
  } else {
    lin_dgrad(G, st, W, LL.qkv, &LL.qkv_A, &LL.qkv_B, dqkv, qkvd, qkvd, G.dh, h, h);
    lora_wgrad(G, st, dW, LL.qkv_A, LL.qkv_B, A.h1, h, h, A.u_qkv, dqkv, qkvd, qkvd, first);
  }
  RP_CUDA(cudaStreamWaitEvent(st, G.ev_dx16_free[xa], 0));  // wgrad(down) read dx_a
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_rmsnorm_bwd(G.dh, A.xin, W + LL.in_norm.off, A.rstd1, G.dx32[1], G.dx32[0], dx_a,
                        full ? dW + LL.in_norm.off : nullptr, T, h, st));
    prof_end(pi_, st, 2, 14.0 * T * h);
  }
  RP_CUDA(cudaEventRecord(A.ev_chain_free, st));
  kernels += 8;
}

// MoE MLP forward (Qwen3-MoE sparse block, modeling_qwen3_moe.py:254-287):
// router logits (fp32) -> softmax / top-k -> expert-sorted rows -> grouped
// gate/up GEMM -> SwiGLU -> grouped down GEMM -> weighted sum + residual.
// A.gu / A.act keep the T*ek sorted rows for the backward.
void Runtime::moe_mlp_fwd(Gpu& G, cudaStream_t st, const uint16_t* W, LayerActs& A,
                          uint16_t* x_out) {
  const int h = s.h, m = s.m, E = s.E, k = s.ek, Tk = T * k;
  gemm(st, A.h2, h, false, W + LL.router.off, h, false, A.r_logits, E, true, false, T, E, h);
  RP_K(rp_moe_route(A.r_logits, T, E, k, s.norm_topk ? 1 : 0, A.r_idx, A.r_w, G.m_counts, st));
  RP_K(rp_moe_permute(A.h2, h, T, h, k, E, A.r_idx, A.r_w, G.m_counts, A.r_off, G.m_cursor,
                      A.r_pos, A.r_ws, G.m_xs, st));
  grouped(st, G.m_xs, h, W + LL.gate_up.off, h, false, A.gu, 2 * m, Tk, 2 * m, h, A.r_off, 2 * m);
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_swiglu_fwd(A.gu, A.act, Tk, m, st));
    prof_end(pi_, st, 2, 6.0 * Tk * m);
  }
  grouped(st, A.act, m, W + LL.down.off, m, false, G.m_ys, h, Tk, h, m, A.r_off, h);
  RP_K(rp_moe_combine(G.m_ys, A.r_pos, A.r_w, T, k, h, A.x2, h, x_out, h, st));
}

// MoE MLP backward with frozen experts and router: G.dh = dL/dh2 from dy =
// dL/d(MLP output) through the weighted expert sum (dw per routed row), the
// experts (grouped dgrad GEMMs, SwiGLU backward) and the router (top-k
// renormalisation + softmax backward, router dgrad GEMM).
void Runtime::moe_mlp_bwd(Gpu& G, cudaStream_t st, const uint16_t* W, LayerActs& A,
                          const uint16_t* dy, uint16_t* dgu) {
  const int h = s.h, m = s.m, E = s.E, k = s.ek, Tk = T * k;
  RP_K(rp_moe_gather(dy, h, T, h, k, A.r_pos, G.m_xs, st));
  grouped(st, G.m_xs, h, W + LL.down.off, m, true, G.m_dact, m, Tk, m, h, A.r_off, h);
  {
    const int pi_ = prof_begin(st);
    RP_K(rp_moe_swiglu_bwd(G.m_dact, A.gu, A.r_ws, Tk, m, dgu, G.m_dws, st));
    prof_end(pi_, st, 2, 10.0 * Tk * m);
  }
  grouped(st, dgu, 2 * m, W + LL.gate_up.off, h, true, G.m_ys, h, Tk, h, 2 * m, A.r_off, 2 * m);
  RP_K(rp_moe_router_bwd(A.r_logits, T, E, k, s.norm_topk ? 1 : 0, A.r_idx, A.r_pos, G.m_dws,
                         G.m_dlogits, st));
  gemm(st, G.m_dlogits, E, false, W + LL.router.off, h, true, G.m_dh32, h, true, false, T, h, E);
  RP_K(rp_moe_combine_bwd(G.m_ys, A.r_pos, T, k, h, G.m_dh32, G.dh, h, st));
  kernels += 5;
}

// Head pseudo-layer: final RMSNorm + LM head + CE forward and backward,
// chunked over token rows: only a [rows, V] logits chunk ever exists, and the
// CE kernel overwrites it in place with dlogits.
void Runtime::head_fwd_bwd(Gpu& G, const uint16_t* x, int gmb, bool first, float grad_scale,
                           cudaStream_t on) {
  DevGroup& D = G.groups[s.L + 1];
  const uint16_t* W = D.w[exec_iter & 1];
  float* dW = D.grad[last_iter & 1];
  cudaStream_t st = on ? on : G.compute;
  // pipelined fused stage: the head runs beside the previous micro-batch's
  // backward, so it uses its own dh and hands its output gradient over in
  // hdx32 / hdx16 (copied into dx32[0] / dx16 by the backward stream)
  const bool piped = on && on != G.compute;
  uint16_t* dh = piped ? G.hdh : G.dh;
  const int h = s.h, V = s.V;
  const bool train = trainable(s.L + 1);  // LoRA: the head is frozen
  if (first && train) {
    grad_free(G, s.L + 1, st);
    RP_CUDA(cudaMemsetAsync(dW + HL.final_norm.off, 0, (size_t)h * 4, st));
  }
  RP_K(rp_rmsnorm_fwd(x, h, W + HL.final_norm.off, G.hN, h, G.rstdN, T, h, (float)s.eps, st));
  const int rows = std::min(T, logits_rows);
  for (int r0 = 0; r0 < T; r0 += rows) {
    const int nr = std::min(rows, T - r0);
    gemm(st, G.hN + (int64_t)r0 * h, h, false, W + HL.lm_head.off, h, false, G.logits, V, false,
         false, nr, V, h);
    {
    const int pi_ = prof_begin(st);
    RP_K(rp_ce_fwd_bwd(G.logits, V, G.labels_dev + (int64_t)gmb * T + r0, nr, V, grad_scale,
                       G.loss_dev, nullptr, st));
    prof_end(pi_, st, 2, 6.0 * nr * (double)V);
  }
    gemm(st, G.logits, V, false, W + HL.lm_head.off, h, true, dh + (int64_t)r0 * h, h, false,
         false, nr, h, V);
    if (train)
      gemm(st, G.logits, V, true, G.hN + (int64_t)r0 * h, h, true, dW + HL.lm_head.off, h, true,
           !(first && r0 == 0), V, h, nr);
    kernels += 1;
  }
  if (piped) {
    RP_CUDA(cudaStreamWaitEvent(st, G.ev_hdx_free, 0));  // previous hand-over consumed
    RP_K(rp_rmsnorm_bwd(dh, x, W + HL.final_norm.off, G.rstdN, nullptr, G.hdx32, G.hdx16,
                        train ? dW + HL.final_norm.off : nullptr, T, h, st));
  } else {
    RP_CUDA(cudaStreamWaitEvent(st, G.ev_dx16_free[G.dx16 == G.dx16s[0] ? 0 : 1], 0));
    RP_K(rp_rmsnorm_bwd(dh, x, W + HL.final_norm.off, G.rstdN, nullptr, G.dx32[0], G.dx16,
                        train ? dW + HL.final_norm.off : nullptr, T, h, st));
  }
  kernels += 2;
}

// ---- one (round, slot) on one worker ----------------------------------------------------
void Runtime::run_slot(Gpu& G, int it, int round, int slot, int first_round, float grad_scale) {
  const roundpipe::StageSlot& ss = slots[slot];
  const int a = ss.layers.first, b = ss.layers.last;
  const int rin = round - first_round;
  const int par = round % parities;
  const bool has_grads = ss.kind != StageKind::Forward;
  cudaStream_t st = G.compute;
  Gpu* next = slot + 1 < S ? &gpus[worker_of(round, slot + 1)] : nullptr;

  // ---- uploads, in the order compute needs the layers
  const std::vector<int> gs = slot_groups(ss);  // groups used by this slot
  for (int g : gs) {
    const bool last_use = rin == R - 1 && (g == 0 ? ss.kind != StageKind::Backward
                                                  : ss.kind != StageKind::Forward);
    upload(G, g, it, last_use);
  }
  auto wait_group = [&](int g) {
    RP_CUDA(cudaStreamWaitEvent(st, G.groups[g].ev_upload[it & 1], 0));
  };
  // groups whose grads this slot produces
  std::vector<int> grad_groups;
  if (has_grads) {
    for (int l = a; l <= std::min(b, s.L - 1); ++l)
      if (trainable(l + 1)) grad_groups.push_back(l + 1);
    if (b == s.L && trainable(s.L + 1)) grad_groups.push_back(s.L + 1);
    if (a == 0 && trainable(0)) grad_groups.push_back(0);
    // grad[t%2] may be overwritten once AdamW consumed it (edge 4, parity form)
    // HBM-resident groups keep ONE grad buffer: they wait last iteration's
    // AdamW right before their first grad write instead (grad_free), so the
    // slot does not stall on the whole resident optimizer pass
    for (int g : grad_groups) {
      DevGroup& D = G.groups[g];
      if (pooled) {  // a fresh slab for this iteration's grads (edge (4) = its free event)
        if (rin > 0) continue;
        const int p = it & 1;
        if (D.grad_slab[p] >= 0) throw RtError(RP_E_INTERNAL, "grad slab still bound");
        D.grad_slab[p] = slab_acquire(G, (std::size_t)host[g].tn() * 4, 1, st);
        const Slab& sl = G.slabs[D.grad_slab[p]];
        D.grad[p] = static_cast<float*>(sl.p) - host[g].t_off;
        if (sl.tag_kind == (int)roundpipe::ActionKind::GradCopy)
          proto_edge(roundpipe::ActionKind::GradCopy, sl.tag_group, sl.tag_iter,
                     roundpipe::ActionKind::GradWrite, g, it);
        continue;
      }
      if (host[g].d_state || D.adam_iter[it & 1] < 0) continue;
      RP_CUDA(cudaStreamWaitEvent(st, D.ev_adam[it & 1], 0));  // edge (4), parity buffers
      proto_edge(roundpipe::ActionKind::GradCopy, g, D.adam_iter[it & 1],
                 roundpipe::ActionKind::GradWrite, g, it);
    }
  }
  RP_CUDA(cudaStreamWaitEvent(st, G.ev_tokens, 0));
  const bool want_tl = cfg.flags & RP_RT_RECORD_TIMELINE;
  const std::size_t Th2 = (std::size_t)T * s.h * 2, Th4 = (std::size_t)T * s.h * 4;

  // Pipelined fused stage (whole model in one slot): forward + head of
  // micro-batch k+1 on `fwd2` beside the backward of k on `compute`.
  // Profiled steps run the plain order so kernel times stay their own.
  if (ss.kind == StageKind::Fused && a == 0 && !G.acts2.empty() && !prof_on) {
    cudaStream_t F = G.fwd2;
    join(G, st, F);  // uploads, tokens, edge-4 waits so far
    auto wait_on = [&](cudaStream_t q, int g) {
      RP_CUDA(cudaStreamWaitEvent(q, G.groups[g].ev_upload[it & 1], 0));
    };
    const int nl = s.L;
    for (int mb = 0; mb < MR; ++mb) {
      const int gmb = rin * MR + mb;
      const bool first = rin == 0 && mb == 0;
      LayerActs* acts = (mb & 1) ? G.acts2.data() : G.acts.data();
      release_window(G);  // next iteration's weights, paced by this micro-batch
      TaskRecord rec{};
      if (want_tl) {
        rec.task = roundpipe::Task{it, round, slot, mb, G.id, ss.dur_ns};
        rec.worker = G.id;
        rec.start = new_event(true);
        rec.end = new_event(true);
        RP_CUDA(cudaEventRecord(rec.start, st));
      }
      // forward + LM head of mb on F
      const int32_t* ids = G.tokens_dev + (int64_t)gmb * T;
      RP_CUDA(cudaStreamWaitEvent(F, acts[0].ev_free, 0));
      RP_CUDA(cudaStreamWaitEvent(F, acts[0].ev_chain_free, 0));
      wait_on(F, 0);
      RP_K(rp_embed_fwd(ids, G.groups[0].w[it & 1], acts[0].x, T, s.h, F));
      ++kernels;
      const uint16_t* x = acts[0].x;
      for (int i = 0; i < nl; ++i) {
        wait_on(F, i + 1);
        uint16_t* out = (i + 1 < nl) ? acts[i + 1].x : G.xbuf[1];
        prof_unit(i, 0);
        layer_fwd(G, i, x, acts[i], out, F);
        x = out;
      }
      wait_on(F, s.L + 1);
      prof_unit(s.L, 3);
      head_fwd_bwd(G, x, gmb, first, grad_scale, F);
      RP_CUDA(cudaEventRecord(G.ev_head_done, F));
      // backward of mb on compute, starting from the head's hand-over
      RP_CUDA(cudaStreamWaitEvent(st, G.ev_head_done, 0));
      RP_CUDA(cudaStreamWaitEvent(st, G.ev_dx16_free[G.dx16 == G.dx16s[0] ? 0 : 1], 0));
      RP_CUDA(cudaMemcpyAsync(G.dx32[0], G.hdx32, Th4, cudaMemcpyDeviceToDevice, st));
      RP_CUDA(cudaMemcpyAsync(G.dx16, G.hdx16, Th2, cudaMemcpyDeviceToDevice, st));
      RP_CUDA(cudaEventRecord(G.ev_hdx_free, st));
      for (int i = nl - 1; i >= 0; --i) {
        prof_unit(i, 1);
        layer_bwd(G, i, acts[i], first);
      }
      if (trainable(0)) {  // embedding gradient (scatter-add of dL/dx_0)
        float* dE = G.groups[0].grad[it & 1];
        if (first) {
          grad_free(G, 0, st);
          RP_CUDA(cudaMemsetAsync(dE, 0, (size_t)s.V * s.h * 4, st));
        }
        RP_K(rp_embed_bwd(ids, G.dx32[0], dE, T, s.h, st));
        ++kernels;
      }
      if (want_tl) {
        RP_CUDA(cudaEventRecord(rec.end, st));
        records.push_back(rec);
      }
    }
  } else
  for (int mb = 0; mb < MR; ++mb) {
    const int gmb = rin * MR + mb;
    const bool first = rin == 0 && mb == 0;
    const int hb = par * MR + mb;  // hand-off buffer index
    release_window(G);  // next iteration's weights, paced by this micro-batch
    TaskRecord rec{};
    if (want_tl) {
      rec.task = roundpipe::Task{it, round, slot, mb, G.id, ss.dur_ns};
      rec.worker = G.id;
      rec.start = new_event(true);
      rec.end = new_event(true);
      RP_CUDA(cudaEventRecord(rec.start, st));
    }
    const int32_t* ids = G.tokens_dev + (int64_t)gmb * T;
    // input activation of the slot (fwd / fused)
    const uint16_t* x_in = nullptr;
    Slotbuf* in_buf = nullptr;
    if (ss.kind != StageKind::Backward) {
      if (a == 0) {
        wait_group(0);
        uint16_t* dst = ss.kind == StageKind::Fused && a < s.L ? G.acts[0].x : G.xbuf[0];
        RP_K(rp_embed_fwd(ids, G.groups[0].w[it & 1], dst, T, s.h, st));
        ++kernels;
        x_in = dst;
      } else {
        in_buf = &G.hand_act[hb];
        RP_CUDA(cudaStreamWaitEvent(st, in_buf->ready, 0));
        x_in = static_cast<const uint16_t*>(in_buf->p);
      }
    }
    if (ss.kind == StageKind::Forward) {
      const uint16_t* x = x_in;
      for (int l = a; l <= b; ++l) {
        // checkpoint x_l for the backward slot that recomputes layer l
        Gpu& O = gpus[worker_of(round, bwd_slot_of[l])];
        Slotbuf& ck = O.ckpt[((std::size_t)par * s.L + l) * MR + mb];
        if (pooled) {  // a slab of the consumer's pool until the recomputing slot read it
          if (ck.slab >= 0) throw RtError(RP_E_INTERNAL, "checkpoint slab still bound");
          ck.slab = slab_acquire(O, Th2, 5, G.act);
          ck.p = O.slabs[ck.slab].p;
        }
        join(G, st, G.act);
        RP_CUDA(cudaStreamWaitEvent(G.act, ck.read, 0));
        d2d(ck.p, O, x, G, Th2, G.act);
        mark_ready(ck, G, G.act);
        wait_group(l + 1);
        uint16_t* out = x == G.xbuf[0] ? G.xbuf[1] : G.xbuf[0];
        RP_CUDA(cudaStreamWaitEvent(st, ck.ready, 0));  // x_l is overwritten next layer
        prof_unit(l, 0);
        layer_fwd(G, l, x, G.acts[0], out);
        x = out;
      }
      if (in_buf) RP_CUDA(cudaEventRecord(in_buf->read, st));
      // hand x_{b+1} to the next slot
      Slotbuf& nb = next->hand_act[hb];
      join(G, st, G.act);
      RP_CUDA(cudaStreamWaitEvent(G.act, nb.read, 0));
      d2d(nb.p, *next, x, G, Th2, G.act);
      mark_ready(nb, G, G.act);
      RP_CUDA(cudaStreamWaitEvent(st, nb.ready, 0));  // xbuf reuse
    } else if (ss.kind == StageKind::Fused) {
      const int nl = s.L - a;  // decoder layers inside the fused stage
      const uint16_t* x = x_in;
      for (int i = 0; i < nl; ++i) {
        const int l = a + i;
        wait_group(l + 1);
        uint16_t* out = (i + 1 < nl) ? G.acts[i + 1].x : G.xbuf[1];
        prof_unit(l, 0);
        layer_fwd(G, l, x, G.acts[i], out);
        x = out;
      }
      wait_group(s.L + 1);
      prof_unit(s.L, 3);
      head_fwd_bwd(G, x, gmb, first, grad_scale);
      for (int i = nl - 1; i >= 0; --i) {
        prof_unit(a + i, 1);
        layer_bwd(G, a + i, G.acts[i], first);
      }
      if (in_buf) RP_CUDA(cudaEventRecord(in_buf->read, st));
    } else {  // Backward: incoming dL/dx_{b+1} from the previous slot
      Slotbuf& gi = G.hand_grad[hb];
      RP_CUDA(cudaStreamWaitEvent(st, gi.ready, 0));
      RP_CUDA(cudaMemcpyAsync(G.dx32[0], gi.p, Th4, cudaMemcpyDeviceToDevice, st));
      RP_CUDA(cudaStreamWaitEvent(st, G.ev_dx16_free[G.dx16 == G.dx16s[0] ? 0 : 1], 0));
      RP_K(rp_f32_to_bf16(G.dx32[0], G.dx16, (int64_t)T * s.h, st));
      ++kernels;
      RP_CUDA(cudaEventRecord(gi.read, st));
      for (int l = b; l >= a; --l) {
        Slotbuf& ck = G.ckpt[((std::size_t)par * s.L + l) * MR + mb];
        RP_CUDA(cudaStreamWaitEvent(st, ck.ready, 0));
        wait_group(l + 1);
        LayerActs& A = G.acts[0];
        prof_unit(l, 2);
        layer_fwd(G, l, static_cast<const uint16_t*>(ck.p), A, G.xbuf[1]);  // recompute
        prof_unit(l, 1);
        layer_bwd(G, l, A, first);
        RP_CUDA(cudaEventRecord(ck.read, st));
        if (pooled) {
          slab_release(G, ck.slab, st);
          ck.slab = -1;
          ck.p = nullptr;
        }
      }
    }
    if (has_grads) {
      if (a == 0) {  // embedding gradient (scatter-add of dL/dx_0)
        if (trainable(0)) {
          float* dE = G.groups[0].grad[it & 1];
          if (first) {
            grad_free(G, 0, st);
            RP_CUDA(cudaMemsetAsync(dE, 0, (size_t)s.V * s.h * 4, st));
          }
          RP_K(rp_embed_bwd(ids, G.dx32[0], dE, T, s.h, st));
          ++kernels;
        }
      } else {  // hand dL/dx_a to the next (backward) slot
        Slotbuf& nb = next->hand_grad[hb];
        join(G, st, G.act);
        RP_CUDA(cudaStreamWaitEvent(G.act, nb.read, 0));
        d2d(nb.p, *next, G.dx32[0], G, Th4, G.act);
        mark_ready(nb, G, G.act);
        RP_CUDA(cudaStreamWaitEvent(st, nb.ready, 0));  // dx32 reuse
      }
    }
    if (want_tl) {
      RP_CUDA(cudaEventRecord(rec.end, st));
      records.push_back(rec);
    }
  }
  // last compute read of the slot's weights; grads complete (GradWrite) once
  // the weight-gradient stream has drained into `compute`
  for (int g : gs) RP_CUDA(cudaEventRecord(G.groups[g].ev_lastuse[it & 1], st));
  if (pooled)  // the worker's last use of this version: its slab goes back to the pool
    for (int g : gs) {
      const auto lu = last_use_task.find((int64_t)G.id * 1000003 + g);
      if (lu == last_use_task.end() || lu->second != (int64_t)round * 1000003 + slot) continue;
      DevGroup& D = G.groups[g];
      const int b = it & 1;
      if (D.w_slab[b] < 0) continue;
      slab_release(G, D.w_slab[b], st);
      D.w_slab[b] = -1;
      D.w[b] = nullptr;
      D.loaded[b] = -1;
    }
  if (has_grads) RP_CUDA(cudaStreamWaitEvent(st, G.ev_wgrad, 0));
  if (has_grads && rin == R - 1)
    for (int g : grad_groups) {
      RP_CUDA(cudaEventRecord(G.groups[g].ev_gradwrite, st));
      grad_owner[g] = G.id;
    }
  if (ss.kind == StageKind::Fused) {
    RP_CUDA(cudaEventRecord(ev_loss[G.id], st));
    fused_worker[G.id] = 1;
  }
}

void Runtime::forward_backward(const int32_t* tokens, const int32_t* labels, float* loss) {
  enqueue_iteration(tokens, labels);
  const float l = wait_loss(last_iter);  // early return: once the fused slots are done
  if (loss) *loss = l;
}

// Enqueue one iteration on all workers and return without waiting (the
// non-blocking form of forward_backward: with S=1 plans on N>1 GPUs the next
// iteration runs on another GPU while this one finishes).
void Runtime::enqueue_iteration(const int32_t* tokens, const int32_t* labels) {
  // ids index the embedding table and the logits row: validate them before
  // anything is enqueued (an out-of-range id would make the gather /
  // scatter-add kernels touch memory outside the table); labels < 0 are ignored
  int64_t n_valid = 0;
  for (int64_t i = 0; i < (int64_t)M * T; ++i) {
    if (tokens[i] < 0 || tokens[i] >= s.V || labels[i] >= s.V)
      throw RtError(RP_E_INPUT, "token id / label out of range at index " + std::to_string(i));
    n_valid += labels[i] >= 0;
  }
  const int it = iter++;
  last_iter = it;
  exec_iter = it;
  ensure_horizon(it);
  const int par = it & 1;
  const float grad_scale = n_valid > 0 ? 1.0f / (float)n_valid : 0.f;
  fused_worker.assign(N, 0);
  for (Gpu& G : gpus) {
    set_dev(G);
    G.tokens_dev = G.tokens_par[par];
    G.labels_dev = G.labels_par[par];
    G.loss_dev = G.loss_par[par];
    // iteration it-2 on this worker is done with this parity's buffers
    RP_CUDA(cudaStreamWaitEvent(G.act, G.ev_iter_done[par], 0));
    RP_CUDA(cudaMemcpyAsync(G.tokens_dev, tokens, (size_t)M * T * 4, cudaMemcpyHostToDevice,
                            G.act));
    RP_CUDA(cudaMemcpyAsync(G.labels_dev, labels, (size_t)M * T * 4, cudaMemcpyHostToDevice,
                            G.act));
    RP_CUDA(cudaMemsetAsync(G.loss_dev, 0, 4, G.act));
    RP_CUDA(cudaEventRecord(G.ev_tokens, G.act));
    h2d_bytes += (int64_t)M * T * 8;
  }
  // async: publish AdamW(it-1)'s result now (p_copy, edge 1: every upload of
  // version `it` was enqueued by the previous iteration's prefetch) and queue
  // the uploads of it+1 behind it (edge 2) BEFORE this iteration's compute.
  // CUDA's launch queue lets the host run only ~1K launches ahead of the GPU,
  // so anything enqueued after the compute walk would only start near the end
  // of the iteration and stall the next one on its weights.
  if (cfg.async_optimizer) {
    for (int g = 0; g < ngroups(); ++g)
      if (pend_owner[g] >= 0) p_copy(g);
    plan_upload_windows(it + 1);
  }
  if (pooled) {  // each worker's last use of each group in this iteration
    last_use_task.clear();
    for (std::size_t i = 0; i < sched.tasks.size(); i += MR) {
      const roundpipe::Task& t = sched.tasks[i];
      if (t.iteration != it) continue;
      for (int g : slot_groups(slots[t.slot]))
        last_use_task[(int64_t)t.gpu * 1000003 + g] = (int64_t)t.round * 1000003 + t.slot;
    }
  }
  // walk the dispatch list of this iteration in emission order
  int first_round = -1;
  for (std::size_t i = 0; i < sched.tasks.size();) {
    const roundpipe::Task& t = sched.tasks[i];
    if (t.iteration < it) {
      ++i;
      continue;
    }
    if (t.iteration > it) break;
    if (first_round < 0) first_round = t.round;
    Gpu& G = gpus[t.gpu];
    set_dev(G);
    run_slot(G, it, t.round, t.slot, first_round, grad_scale);
    i += MR;  // a (round, slot) is MR consecutive tasks on one worker
  }
  flush_windows();  // every upload of it+1 is enqueued before p_copy(it+1) (edge 1)
  for (Gpu& G : gpus) {  // this parity's buffers are free once `compute` gets here
    set_dev(G);
    RP_CUDA(cudaEventRecord(G.ev_iter_done[par], G.compute));
    if (fused_worker[G.id]) {
      RP_CUDA(cudaStreamWaitEvent(G.act, ev_loss[G.id], 0));
      RP_CUDA(cudaMemcpyAsync(loss_host + par * N + G.id, G.loss_dev, 4, cudaMemcpyDeviceToHost,
                              G.act));
      RP_CUDA(cudaEventRecord(G.ev_loss_par[par], G.act));
      flags.set(G.act, flag_loss(G.id), (uint32_t)it + 1);  // loss of `it` is on the host
    }
  }
  fused_par[par] = fused_worker;
  grad_scale_par[par] = grad_scale;
  iter_par[par] = it;
  grads_pending = true;
}

// Mean token loss of iteration `it` (one of the last two enqueued).
float Runtime::wait_loss(int it) {
  const int par = it & 1;
  if (it < 0 || iter_par[par] != it)
    throw RtError(RP_E_INPUT, "loss of iteration " + std::to_string(it) + " is no longer held");
  // early return: the controller polls the workers' loss flag
  // words instead of blocking in the driver; every ~1K polls it checks the
  // loss event for a device error so a failed step cannot spin forever
  double total = 0.0;
  for (Gpu& G : gpus) {
    if (!fused_par[par][G.id]) continue;
    for (long spins = 0; flags.read(flag_loss(G.id)) < (uint32_t)it + 1; ++spins) {
      if (spins % 1024 == 1023) {
        set_dev(G);
        const cudaError_t e = cudaEventQuery(G.ev_loss_par[par]);
        if (e != cudaSuccess && e != cudaErrorNotReady) RP_CUDA(e);
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    total += static_cast<volatile float*>(loss_host)[par * N + G.id];
  }
  return (float)(total * grad_scale_par[par]);
}

// ---- optimizer lane -------------------------------------------------------------------
// AdamW for one parameter group over fp32 state chunks streamed from pinned
// host memory: H2D (opt_h2d) -> kernel (opt_comp) -> D2H (opt_d2h), two chunk
// slots in flight. Consumes grad[parity] (g_copy) and leaves the new bf16
// weights in `pend` for p_copy.
void Runtime::adam_group(Gpu& G, int g, int parity) {
  DevGroup& D = G.groups[g];
  HostGroup& H = host[g];
  const int step_no = ++H.step;
  RP_CUDA(cudaStreamWaitEvent(G.opt_comp, D.ev_gradwrite, 0));  // edge (3)
  proto_edge(roundpipe::ActionKind::GradWrite, g, last_iter, roundpipe::ActionKind::GradCopy, g,
             last_iter);
  D.adam_iter[parity] = last_iter;
  RP_CUDA(cudaStreamWaitEvent(G.opt_comp, D.ev_pcopy, 0));      // pend free again
  if (H.d_state) {  // HBM-resident fp32 state: one fused pass, no PCIe
    cudaStream_t q = G.opt_res;
    RP_CUDA(cudaStreamWaitEvent(q, D.ev_gradwrite, 0));  // edge (3)
    RP_CUDA(cudaStreamWaitEvent(q, D.ev_pcopy, 0));      // pend free again
    // the shared d_state was last updated by another logical worker's
    // optimizer stream (grads land on a different worker each iteration)
    if (state_ev[g]) RP_CUDA(cudaStreamWaitEvent(q, state_ev[g], 0));
    cudaEvent_t xa = xfer_begin(q);
    const int pi_ = prof_begin(q);
    const int64_t tn = H.tn(), to = H.t_off;
    // direct: the result is version last+2 (async, staleness 1) or last+1
    // (sync); it overwrites the device buffer of version last (resp. last-1)
    // once that version's last compute read is done
    const int ver = last_iter + (cfg.async_optimizer ? 2 : 1), b = ver & 1;
    uint16_t* out = D.pend;
    if (H.direct) {
      RP_CUDA(cudaStreamWaitEvent(q, D.ev_lastuse[b], 0));  // WAR on w[b]
      // a copy-in of w[b] still in flight (e.g. the version resumed from a checkpoint)
      RP_CUDA(cudaStreamWaitEvent(q, D.ev_upload[b], 0));
      out = D.w[b];
      if (to > 0 && D.loaded[b] < 0)  // frozen part (LoRA base) never written to w[b] yet
        RP_CUDA(cudaMemcpyAsync(D.w[b], H.w16, to * 2, cudaMemcpyHostToDevice, q));
    }
    RP_K(rp_adamw(H.d_state, H.d_state + tn, H.d_state + 2 * tn, D.grad[parity] + to, out + to,
                  tn, &cfg.adam, step_no, q));
    prof_end(pi_, q, 3, 30.0 * tn);
    ++kernels;
    RP_CUDA(cudaEventRecord(D.ev_adam[parity], q));
    if (!D.ev_state) D.ev_state = new_event(false);
    RP_CUDA(cudaEventRecord(D.ev_state, q));
    state_ev[g] = D.ev_state;
    xfer_end(xa, q, 2, g - 1, last_iter, G.id);
    H.host_stale = true;
    if (H.direct) {  // published in place: no p_copy, no upload
      RP_CUDA(cudaEventRecord(D.ev_upload[b], q));
      flags.set(q, flag_pub(g), (uint32_t)ver);  // = the ParamCopy index (ver - 1) + 1
      D.loaded[b] = ver;
      H.w16_stale = true;
      return;
    }
    pend_owner[g] = G.id;
    if (!cfg.async_optimizer) p_copy(g);
    return;
  }
  if (pooled && !D.pend) {  // AdamW output slab until p_copy publishes it
    D.pend_slab = slab_acquire(G, (std::size_t)H.tn() * 2, 2, G.opt_comp);
    D.pend = static_cast<uint16_t*>(G.slabs[D.pend_slab].p) - H.t_off;
  }
  if (state_ev[g]) RP_CUDA(cudaStreamWaitEvent(G.opt_h2d, state_ev[g], 0));  // prev. write-back
  // in-place publication (one worker): version `ver` overwrites w[b] once
  // iteration ver-2's (sync: ver-1's) last compute read of it is done
  const int ver = last_iter + (cfg.async_optimizer ? 2 : 1), vb = ver & 1;
  uint16_t* out = D.pend;
  if (H.direct) {
    RP_CUDA(cudaStreamWaitEvent(G.opt_comp, D.ev_lastuse[vb], 0));  // WAR on w[vb]
    RP_CUDA(cudaStreamWaitEvent(G.opt_comp, D.ev_upload[vb], 0));
    out = D.w[vb];
    if (H.t_off > 0 && D.loaded[vb] < 0)  // frozen part (LoRA base) never written to w[vb] yet
      RP_CUDA(cudaMemcpyAsync(D.w[vb], H.w16, H.t_off * 2, cudaMemcpyHostToDevice, G.opt_comp));
  }
  cudaEvent_t xa = xfer_begin(G.opt_h2d);
  for (int64_t off = H.t_off; off < H.n; off += chunk_elems) {  // trainable region
    const int64_t n = std::min<int64_t>(chunk_elems, H.n - off);
    const int sl = G.opt_slot;
    G.opt_slot = (G.opt_slot + 1) % Gpu::kOptSlots;
    float** buf = G.opt_buf[sl];
    RP_CUDA(cudaStreamWaitEvent(G.opt_h2d, G.opt_free[sl], 0));
    RP_CUDA(cudaMemcpyAsync(buf[0], H.master + off, n * 4, cudaMemcpyHostToDevice, G.opt_h2d));
    RP_CUDA(cudaMemcpyAsync(buf[1], H.m + off, n * 4, cudaMemcpyHostToDevice, G.opt_h2d));
    RP_CUDA(cudaMemcpyAsync(buf[2], H.v + off, n * 4, cudaMemcpyHostToDevice, G.opt_h2d));
    h2d_bytes += n * 12;
    join(G, G.opt_h2d, G.opt_comp);
    const int pi_ = prof_begin(G.opt_comp);
    RP_K(rp_adamw(buf[0], buf[1], buf[2], D.grad[parity] + off, out + off, n, &cfg.adam,
                  step_no, G.opt_comp));
    prof_end(pi_, G.opt_comp, 3, 30.0 * n);
    ++kernels;
    join(G, G.opt_comp, G.opt_d2h);
    RP_CUDA(cudaMemcpyAsync(H.master + off, buf[0], n * 4, cudaMemcpyDeviceToHost, G.opt_d2h));
    RP_CUDA(cudaMemcpyAsync(H.m + off, buf[1], n * 4, cudaMemcpyDeviceToHost, G.opt_d2h));
    RP_CUDA(cudaMemcpyAsync(H.v + off, buf[2], n * 4, cudaMemcpyDeviceToHost, G.opt_d2h));
    d2h_bytes += n * 12;
    RP_CUDA(cudaEventRecord(G.opt_free[sl], G.opt_d2h));
  }
  RP_CUDA(cudaEventRecord(D.ev_adam[parity], G.opt_comp));  // g_copy(l, t) complete
  if (pooled) {  // grads consumed: the slab goes back to the pool
    slab_release(G, D.grad_slab[parity], G.opt_comp, (int)roundpipe::ActionKind::GradCopy, g,
                 last_iter);
    D.grad_slab[parity] = -1;
    D.grad[parity] = nullptr;
  }
  if (!D.ev_state) D.ev_state = new_event(false);
  RP_CUDA(cudaEventRecord(D.ev_state, G.opt_d2h));
  xfer_end(xa, G.opt_d2h, 2, g - 1, last_iter, G.id);
  state_ev[g] = D.ev_state;
  if (H.direct) {  // published in place: no p_copy, no upload
    RP_CUDA(cudaEventRecord(D.ev_upload[vb], G.opt_comp));
    flags.set(G.opt_comp, flag_pub(g), (uint32_t)ver);  // = the ParamCopy index (ver - 1) + 1
    D.loaded[vb] = ver;
    H.w16_stale = true;
    return;
  }
  pend_owner[g] = G.id;
  if (!cfg.async_optimizer) p_copy(g);  // sync: iteration t+1 sees grads of t
}

void Runtime::step() {
  if (!grads_pending) return;
  grads_pending = false;
  const int parity = last_iter & 1;
  // optimizer lane order. async: GradWrite order (head first, then layers
  // L-1..0) — the result is needed only two iterations later. sync: the
  // next iteration's forward order (embedding, layers 0..L-1, head): every
  // GradWrite lands within the last micro-batch's backward, and per-layer
  // publication then lets iteration t+1's first layers start while the
  // deeper layers' AdamW still streams
  std::vector<int> order;
  if (cfg.async_optimizer) {
    order.push_back(s.L + 1);
    for (int l = s.L - 1; l >= 0; --l) order.push_back(l + 1);
    order.push_back(0);
  } else {
    for (int g = 0; g < ngroups(); ++g) order.push_back(g);
  }
  for (int g : order) {
    if (!trainable(g)) continue;  // frozen (LoRA base): no grads, no optimizer
    Gpu& G = gpus[grad_owner[g]];
    set_dev(G);
    adam_group(G, g, parity);
  }
  // sync: uploads of t+1 follow each group's publication, in the same order
  if (!cfg.async_optimizer) prefetch(last_iter + 1);
  if (event_pool.size() > 500000) sync_all();
}

void Runtime::sync_all() {
  for (Gpu& G : gpus) {
    set_dev(G);
    RP_CUDA(cudaDeviceSynchronize());
  }
}

// Releases every device allocation (weights, grads, activations, hand-off
// and checkpoint buffers, scratch, the optimizer ring, resident state), the
// per-stream kernel workspaces, events and streams, so a new runtime in the
// same process (e.g. a re-plan on measured costs) starts from a clean device.
Runtime::~Runtime() {
  for (Gpu& G : gpus) {
    cudaSetDevice(G.dev);
    cudaDeviceSynchronize();
  }
  for (auto e : event_pool) cudaEventDestroy(e);
  for (Gpu& G : gpus) {
    cudaSetDevice(G.dev);
    for (cudaStream_t st : {G.compute, G.act, G.wgrad, G.w_h2d, G.opt_h2d, G.opt_d2h, G.opt_comp,
                            G.opt_res, G.fwd2})
      if (st) {
        release_stream_workspaces(st);
        cudaStreamDestroy(st);
      }
    for (void* p : G.owned) cudaFree(p);
    G.owned.clear();
  }
  if (loss_host) cudaFreeHost(loss_host);
  if (!gpus.empty()) cudaSetDevice(gpus[0].dev);
  for (auto& H : host)
    if (H.d_state) cudaFree(H.d_state);
}

}  // namespace rt
}  // namespace rp

// ======================================================================== C-ABI
namespace {
using rp::rt::RtError;
using rp::rt::Runtime;
thread_local std::string g_rt_error;

template <class F>
int rt_guard(F&& f) {
  try {
    g_rt_error.clear();
    f();
    return RP_OK;
  } catch (const RtError& e) {
    g_rt_error = e.what();
    return e.code;
  } catch (const roundpipe::InfeasibleError& e) {
    g_rt_error = e.what();
    return RP_E_INFEASIBLE;
  } catch (const roundpipe::ConfigError& e) {
    g_rt_error = e.what();
    return RP_E_INPUT;
  } catch (const std::invalid_argument& e) {
    g_rt_error = e.what();
    return RP_E_INPUT;
  } catch (const std::exception& e) {
    g_rt_error = e.what();
    return RP_E_INTERNAL;
  }
}

uint16_t f32_to_bf16_host(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
float bf16_to_f32_host(uint16_t b) {
  const uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
Runtime* R(rp_runtime_t* p) { return reinterpret_cast<Runtime*>(p); }
int gidx(Runtime* rt, int32_t group) {
  if (group < -1 || group > rt->s.L) throw RtError(RP_E_INPUT, "parameter group out of range");
  return group + 1;
}
}  // namespace

#define RP_API extern "C" __attribute__((visibility("default")))

RP_API const char* rp_runtime_last_error(void) { return g_rt_error.c_str(); }

RP_API int rp_runtime_create(const rp_runtime_config_t* cfg, rp_runtime_t** out) {
  return rt_guard([&] {
    if (!cfg || !out) throw RtError(RP_E_INPUT, "null argument");
    auto rt = std::make_unique<Runtime>();
    rt->init(*cfg);
    *out = reinterpret_cast<rp_runtime_t*>(rt.release());
  });
}

RP_API int rp_runtime_destroy(rp_runtime_t* rt) {
  return rt_guard([&] { delete R(rt); });
}

RP_API int rp_runtime_plan(rp_runtime_t* p, rp_stage_plan_t* plan, int64_t* slot_durs,
                           int32_t cap, int32_t* n_slots) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    const auto& pl = rt->plan;
    if (plan) {
      plan->num_fwd = (int32_t)pl.fwd_stages.size();
      plan->num_bwd = (int32_t)pl.bwd_stages.size();
      plan->fused = rp_layer_range_t{pl.fused_stage.first, pl.fused_stage.last};
      plan->t_max_ns = pl.t_max_ns;
      plan->objective = pl.objective;
      if (plan->num_fwd > plan->cap || plan->num_bwd > plan->cap)
        throw RtError(RP_E_TOOSMALL, "plan capacity");
      for (int i = 0; i < plan->num_fwd; ++i)
        plan->fwd[i] = rp_layer_range_t{pl.fwd_stages[i].first, pl.fwd_stages[i].last};
      for (int i = 0; i < plan->num_bwd; ++i)
        plan->bwd[i] = rp_layer_range_t{pl.bwd_stages[i].first, pl.bwd_stages[i].last};
    }
    if (n_slots) *n_slots = (int32_t)rt->slots.size();
    if (slot_durs) {
      if ((int32_t)rt->slots.size() > cap) throw RtError(RP_E_TOOSMALL, "slot capacity");
      for (std::size_t i = 0; i < rt->slots.size(); ++i) slot_durs[i] = rt->slots[i].dur_ns;
    }
  });
}

RP_API int rp_runtime_costs(rp_runtime_t* p, rp_layer_cost_t* out, int32_t cap, int32_t* n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    *n = (int32_t)rt->costs.size();
    if (*n > cap) throw RtError(RP_E_TOOSMALL, "cost capacity");
    for (int i = 0; i < *n; ++i)
      out[i] = rp_layer_cost_t{rt->costs[i].t_fwd_ns, rt->costs[i].t_bwd_ns,
                               rt->costs[i].param_bytes, rt->costs[i].act_ckpt_bytes,
                               rt->costs[i].act_full_bytes};
  });
}

RP_API int rp_param_count(rp_runtime_t* p, int32_t group, int64_t* n) {
  return rt_guard([&] { *n = R(p)->group_numel(gidx(R(p), group)); });
}

// Flat layout of a group: (offset, rows, cols) per tensor, in the order
// embed | in_norm qkv q_norm k_norm o post_norm [router] gate_up down | final_norm lm_head.
RP_API int rp_param_layout(rp_runtime_t* p, int32_t group, int64_t* offs, int64_t* rows,
                           int64_t* cols, int32_t cap, int32_t* n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    const int g = gidx(rt, group);
    std::vector<rp::rt::Tensor> ts;
    if (g == 0) ts = {rp::rt::Tensor{0, rt->s.V, rt->s.h}};
    else if (g == rt->s.L + 1) ts = {rt->HL.final_norm, rt->HL.lm_head};
    else {
      const auto& L = rt->LL;
      ts = {L.in_norm, L.qkv, L.q_norm, L.k_norm, L.o, L.post_norm};
      if (rt->s.moe()) ts.push_back(L.router);
      ts.push_back(L.gate_up);
      ts.push_back(L.down);
      if (rt->lora_r)  // adapters after the base tensors (MoE: attention only)
        for (const auto* t : {&L.qkv_A, &L.qkv_B, &L.o_A, &L.o_B, &L.gu_A, &L.gu_B, &L.down_A,
                              &L.down_B})
          if (t->numel() > 0) ts.push_back(*t);
    }
    *n = (int32_t)ts.size();
    if (*n > cap) throw RtError(RP_E_TOOSMALL, "layout capacity");
    for (int i = 0; i < *n; ++i) {
      offs[i] = ts[i].off;
      rows[i] = ts[i].rows;
      cols[i] = ts[i].cols;
    }
  });
}

RP_API int rp_set_params(rp_runtime_t* p, int32_t group, const float* values, int64_t n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    const int g = gidx(rt, group);
    rp::rt::HostGroup& H = rt->host[g];
    if (n != H.n || !values) throw RtError(RP_E_INPUT, "size mismatch");
    rt->sync_all();
    for (int64_t i = 0; i < n; ++i) H.w16[i] = f32_to_bf16_host(values[i]);
    for (int64_t i = H.t_off; i < n; ++i) {  // trainable region (all of it unless LoRA)
      H.master[i] = values[i];
      H.m[i] = 0.f;
      H.v[i] = 0.f;
    }
    H.step = 0;
    H.host_stale = false;
    H.w16_stale = false;
    rt->push_resident(g);
    for (auto& G : rt->gpus) G.groups[g].loaded[0] = G.groups[g].loaded[1] = -1;
    // a pending staleness-1 update was computed from the old values: drop it
    // (pending gradients stay and are applied by the next step(), as an
    // optimizer applies .grad to whatever the parameters hold)
    rt->pend_owner[g] = -1;
    rt->uploaders[g].clear();
  });
}

RP_API int rp_get_params(rp_runtime_t* p, int32_t group, int32_t which, float* out, int64_t n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    const int g = gidx(rt, group);
    rp::rt::HostGroup& H = rt->host[g];
    if (n != H.n || !out) throw RtError(RP_E_INPUT, "size mismatch");
    rt->sync_all();
    rt->pull_resident(g);
    rt->pull_w16(g);
    // frozen parts (LoRA base): master = the bf16 weights, grads / m / v = 0
    const int64_t o = H.t_off;
    switch (which) {
      case 0:
        for (int64_t i = 0; i < o; ++i) out[i] = bf16_to_f32_host(H.w16[i]);
        if (n > o) std::memcpy(out + o, H.master + o, (n - o) * 4);
        break;
      case 1:
        for (int64_t i = 0; i < n; ++i) out[i] = bf16_to_f32_host(H.w16[i]);
        break;
      case 2: {
        if (rt->last_iter < 0) throw RtError(RP_E_INPUT, "no iteration has run");
        std::memset(out, 0, o * 4);
        if (n > o) {
          rp::rt::Gpu& G = rt->gpus[rt->grad_owner[g]];
          rt->set_dev(G);
          if (!G.groups[g].grad[rt->last_iter & 1])
            throw RtError(RP_E_INPUT, "gradients already consumed by step() (pooled workers)");
          RP_CUDA(cudaMemcpy(out + o, G.groups[g].grad[rt->last_iter & 1] + o, (n - o) * 4,
                             cudaMemcpyDeviceToHost));
        }
        break;
      }
      case 3:
      case 4:
        std::memset(out, 0, o * 4);
        if (n > o) std::memcpy(out + o, (which == 3 ? H.m : H.v) + o, (n - o) * 4);
        break;
      default: throw RtError(RP_E_INPUT, "bad selector");
    }
  });
}

// ---- host-state checkpoint / resume ------------------------------------------------
// File: "RPCKPT01", int32 {L, h, nq, nk, m, V, ngroups, async}, then per group
// {int64 n, int32 step, int32 pending}, then per group the fp32 master, m, v
// and the bf16 master the GPUs upload. In async mode a group whose AdamW
// result still waits for its p_copy (staleness 1: the next iteration uploads
// the OLD bf16 master) is saved as pending; the pending bf16 weights are
// bf16(fp32 master) by construction (adamw_kernel), so resume re-creates them.
namespace {
constexpr char kCkptMagic[8] = {'R', 'P', 'C', 'K', 'P', 'T', '0', '2'};
struct FileCloser {
  void operator()(FILE* f) const { if (f) std::fclose(f); }
};
void xwrite(FILE* f, const void* p, std::size_t n) {
  if (n && std::fwrite(p, 1, n, f) != n) throw RtError(RP_E_INTERNAL, "checkpoint write failed");
}
void xread(FILE* f, void* p, std::size_t n) {
  if (n && std::fread(p, 1, n, f) != n) throw RtError(RP_E_INPUT, "checkpoint truncated");
}
}  // namespace

RP_API int rp_runtime_save(rp_runtime_t* p, const char* path) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    if (!path) throw RtError(RP_E_INPUT, "null path");
    rt->sync_all();
    for (int g = 0; g < rt->ngroups(); ++g) {
      rt->pull_resident(g);
      rt->pull_w16(g);
    }
    std::unique_ptr<FILE, FileCloser> f(std::fopen(path, "wb"));
    if (!f) throw RtError(RP_E_INPUT, std::string("cannot open ") + path);
    const int ng = rt->ngroups();
    const int32_t hdr[8] = {rt->s.L, rt->s.h, rt->s.nq, rt->s.nk, rt->s.m, rt->s.V, ng,
                            rt->cfg.async_optimizer};
    xwrite(f.get(), kCkptMagic, 8);
    xwrite(f.get(), hdr, sizeof(hdr));
    for (int g = 0; g < ng; ++g) {
      const int64_t n = rt->host[g].n, to = rt->host[g].t_off;
      // pending staleness-1 update: in pend (streamed) or, for a direct group,
      // already in the device buffer of the iteration after next
      const auto& D0 = rt->gpus[0].groups[g];
      const bool direct_pending = rt->host[g].direct && rt->cfg.async_optimizer &&
                                  D0.loaded[(rt->iter + 1) & 1] == rt->iter + 1;
      const int32_t st[2] = {rt->host[g].step, (rt->pend_owner[g] >= 0 || direct_pending) ? 1 : 0};
      xwrite(f.get(), &n, 8);
      xwrite(f.get(), &to, 8);
      xwrite(f.get(), st, 8);
    }
    for (int g = 0; g < ng; ++g) {  // fp32 state of the trainable region, bf16 of all
      const auto& H = rt->host[g];
      if (H.tn() > 0) {
        xwrite(f.get(), H.master + H.t_off, H.tn() * 4);
        xwrite(f.get(), H.m + H.t_off, H.tn() * 4);
        xwrite(f.get(), H.v + H.t_off, H.tn() * 4);
      }
      xwrite(f.get(), H.w16, H.n * 2);
    }
  });
}

RP_API int rp_runtime_load(rp_runtime_t* p, const char* path) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    if (!path) throw RtError(RP_E_INPUT, "null path");
    rt->sync_all();
    std::unique_ptr<FILE, FileCloser> f(std::fopen(path, "rb"));
    if (!f) throw RtError(RP_E_INPUT, std::string("cannot open ") + path);
    char magic[8];
    int32_t hdr[8];
    xread(f.get(), magic, 8);
    xread(f.get(), hdr, sizeof(hdr));
    const int ng = rt->ngroups();
    if (std::memcmp(magic, kCkptMagic, 8) || hdr[0] != rt->s.L || hdr[1] != rt->s.h ||
        hdr[2] != rt->s.nq || hdr[3] != rt->s.nk || hdr[4] != rt->s.m || hdr[5] != rt->s.V ||
        hdr[6] != ng)
      throw RtError(RP_E_INPUT, "checkpoint does not match this model");
    std::vector<int32_t> steps(ng), pending(ng);
    for (int g = 0; g < ng; ++g) {
      int64_t n, to;
      int32_t st[2];
      xread(f.get(), &n, 8);
      xread(f.get(), &to, 8);
      xread(f.get(), st, 8);
      if (n != rt->host[g].n || to != rt->host[g].t_off)
        throw RtError(RP_E_INPUT, "checkpoint group size / trainable region mismatch");
      steps[g] = st[0];
      pending[g] = st[1];
    }
    if (!rt->cfg.async_optimizer)
      for (int g = 0; g < ng; ++g)
        if (pending[g]) throw RtError(RP_E_INPUT, "async checkpoint loaded into a sync runtime");
    for (int g = 0; g < ng; ++g) {
      auto& H = rt->host[g];
      if (H.tn() > 0) {
        xread(f.get(), H.master + H.t_off, H.tn() * 4);
        xread(f.get(), H.m + H.t_off, H.tn() * 4);
        xread(f.get(), H.v + H.t_off, H.tn() * 4);
      }
      xread(f.get(), H.w16, H.n * 2);
      H.step = steps[g];
      H.host_stale = false;
      rt->push_resident(g);
    }
    // device caches hold stale versions; pending AdamW outputs are re-created
    for (auto& G : rt->gpus)
      for (auto& D : G.groups) D.loaded[0] = D.loaded[1] = -1;
    std::vector<uint16_t> tmp;
    for (int g = 0; g < ng; ++g) {
      rt->pend_owner[g] = -1;
      auto& H = rt->host[g];
      H.w16_stale = false;
      if (!pending[g]) continue;
      rp::rt::Gpu& G = rt->gpus[0];
      rt->set_dev(G);
      tmp.resize((std::size_t)H.tn());
      for (int64_t i = H.t_off; i < H.n; ++i)
        tmp[(std::size_t)(i - H.t_off)] = f32_to_bf16_host(H.master[i]);
      if (H.direct) {  // version iter+1: frozen part from the host copy, update on top
        auto& D = G.groups[g];
        const int b = (rt->iter + 1) & 1;
        RP_CUDA(cudaMemcpy(D.w[b], H.w16, H.n * 2, cudaMemcpyHostToDevice));
        RP_CUDA(cudaMemcpy(D.w[b] + H.t_off, tmp.data(), H.tn() * 2, cudaMemcpyHostToDevice));
        D.loaded[b] = rt->iter + 1;
        continue;
      }
      if (rt->pooled && !G.groups[g].pend) {
        G.groups[g].pend_slab = rt->slab_acquire(G, (std::size_t)H.tn() * 2, 2, G.opt_d2h);
        G.groups[g].pend = static_cast<uint16_t*>(G.slabs[G.groups[g].pend_slab].p) - H.t_off;
      }
      RP_CUDA(cudaMemcpy(G.groups[g].pend + H.t_off, tmp.data(), H.tn() * 2,
                         cudaMemcpyHostToDevice));
      rt->pend_owner[g] = 0;
    }
    rt->grads_pending = false;
    // the next iteration runs on the restored bf16 master: queue its uploads
    // now, ahead of the p_copy that will publish the pending update (edge 1)
    rt->prefetch(rt->iter);
  });
}

RP_API int rp_forward_backward(rp_runtime_t* p, const int32_t* tokens, const int32_t* labels,
                               float* loss) {
  return rt_guard([&] {
    if (!tokens || !labels) throw RtError(RP_E_INPUT, "null tokens/labels");
    R(p)->forward_backward(tokens, labels, loss);
  });
}

RP_API int rp_forward_backward_async(rp_runtime_t* p, const int32_t* tokens,
                                     const int32_t* labels, int32_t* iteration) {
  return rt_guard([&] {
    if (!tokens || !labels) throw RtError(RP_E_INPUT, "null tokens/labels");
    R(p)->enqueue_iteration(tokens, labels);
    if (iteration) *iteration = R(p)->last_iter;
  });
}

RP_API int rp_loss(rp_runtime_t* p, int32_t iteration, float* loss) {
  return rt_guard([&] {
    if (!loss) throw RtError(RP_E_INPUT, "null loss");
    *loss = R(p)->wait_loss(iteration);
  });
}

RP_API int rp_step(rp_runtime_t* p) {
  return rt_guard([&] { R(p)->step(); });
}

RP_API int rp_sync(rp_runtime_t* p) {
  return rt_guard([&] { R(p)->sync_all(); });
}

RP_API int rp_timeline(rp_runtime_t* p, rp_timed_event_t* out, int64_t cap, int64_t* n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    rt->sync_all();
    *n = (int64_t)rt->records.size();
    if (*n > cap) throw RtError(RP_E_TOOSMALL, "timeline capacity");
    // one clock per physical device: the anchor of its lowest worker
    std::vector<cudaEvent_t> anchor(rt->ndev, nullptr);
    for (auto& G : rt->gpus)
      if (!anchor[G.dev]) anchor[G.dev] = G.anchor;
    for (int64_t i = 0; i < *n; ++i) {
      const auto& r = rt->records[(std::size_t)i];
      const int dev = rt->gpus[r.worker].dev;
      float a = 0.f, b = 0.f;
      RP_CUDA(cudaEventElapsedTime(&a, anchor[dev], r.start));
      RP_CUDA(cudaEventElapsedTime(&b, anchor[dev], r.end));
      rp_timed_event_t e{};
      e.task.iteration = r.task.iteration;
      e.task.round = r.task.round;
      e.task.slot = r.task.slot;
      e.task.mb = r.task.mb;
      e.task.gpu = r.task.gpu;
      e.start_ns = (int64_t)std::llround((double)a * 1e6);
      e.end_ns = (int64_t)std::llround((double)b * 1e6);
      e.task.dur_ns = e.end_ns - e.start_ns;
      out[i] = e;
    }
  });
}

RP_API int rp_timeline_clear(rp_runtime_t* p) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    rt->sync_all();
    rt->records.clear();
    rt->xfers.clear();
  });
}

RP_API int rp_runtime_stats(rp_runtime_t* p, rp_runtime_stats_t* st) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    std::memset(st, 0, sizeof(*st));
    st->num_layers = rt->s.L;
    st->num_slots = (int32_t)rt->slots.size();
    for (int g = 0; g < rt->ngroups(); ++g) st->params_total += rt->host[g].n;
    st->host_bytes_pinned = (int64_t)rt->arena.size();
    for (auto& G : rt->gpus)
      for (int c = 0; c < 8 && c < (int)G.allocated.size(); ++c)
        st->device_bytes[c] += (int64_t)G.allocated[c];
    st->h2d_bytes = rt->h2d_bytes;
    st->d2h_bytes = rt->d2h_bytes;
    st->p2p_bytes = rt->p2p_bytes;
    st->iterations_done = rt->iter;
    st->kernels_launched = (int32_t)rt->kernels;
    st->resident_params = rt->resident_params;
    for (auto& G : rt->gpus) {
      st->pool_peak_bytes = std::max<int64_t>(st->pool_peak_bytes, (int64_t)G.pool_peak);
      st->pool_bytes += (int64_t)G.pool_bytes;
    }
  });
}

RP_API int rp_runtime_profile(rp_runtime_t* p, int32_t enable) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    rt->sync_all();
    rt->prof_on = enable != 0;
    rt->prof.clear();
    rt->prof_next = 0;
  });
}

// Per category (0 GEMM, 1 attention, 2 HBM-bound stage kernels, 3 AdamW):
// summed kernel time (ms), algorithmic work (FLOPs or bytes), launch count.
RP_API int rp_runtime_profile_read(rp_runtime_t* p, double* time_ms, double* work,
                                   int64_t* launches) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    rt->sync_all();
    for (int c = 0; c < 4; ++c) time_ms[c] = work[c] = 0.0, launches[c] = 0;
    for (const auto& r : rt->prof) {
      float ms = 0.f;
      RP_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      time_ms[r.cat] += ms;
      work[r.cat] += r.work;
      launches[r.cat] += 1;
    }
  });
}

// Measured cost table: per decoder layer the mean kernel time
// of one micro-batch's forward (t_fwd) and of forward + backward (t_bwd, the
// reference's fused/backward stage unit, cost_model.hpp:194), from the
// profiled steps; the head row is the LM-head+CE kernel time (t_bwd = all
// of it, t_fwd = a third: the logits GEMM is one of its three GEMMs). Byte columns come from the cost
// model. Layers without samples keep the cost model's row.
RP_API int rp_runtime_measured_costs(rp_runtime_t* p, rp_layer_cost_t* out, int32_t cap,
                                     int32_t* n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    rt->sync_all();
    const int L = rt->s.L;
    *n = L + 1;
    if (*n > cap) throw RtError(RP_E_TOOSMALL, "cost capacity");
    // per call instance: (unit, summed kernel ns)
    std::vector<std::pair<int, double>> inst;
    for (const auto& r : rt->prof) {
      if (r.lane == 1 || r.unit < 0) continue;  // compute + weight-gradient lanes
      if ((int)inst.size() <= r.inst) inst.resize(r.inst + 1, {-1, 0.0});
      float ms = 0.f;
      RP_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      inst[r.inst].first = r.unit;
      inst[r.inst].second += (double)ms * 1e6;
    }
    std::vector<double> sum((L + 1) * 4, 0.0), cnt((L + 1) * 4, 0.0);
    for (const auto& [u, ns] : inst)
      if (u >= 0 && u < (L + 1) * 4) sum[u] += ns, cnt[u] += 1;
    for (int l = 0; l <= L; ++l) {
      rp_layer_cost_t c{rt->costs[l].t_fwd_ns, rt->costs[l].t_bwd_ns, rt->costs[l].param_bytes,
                        rt->costs[l].act_ckpt_bytes, rt->costs[l].act_full_bytes};
      if (l < L) {
        const double nf = cnt[l * 4 + 0] + cnt[l * 4 + 2], nb = cnt[l * 4 + 1];
        if (nf > 0 && nb > 0) {
          const double tf = (sum[l * 4 + 0] + sum[l * 4 + 2]) / nf;
          c.t_fwd_ns = (int64_t)std::llround(tf);
          c.t_bwd_ns = (int64_t)std::llround(tf + sum[l * 4 + 1] / nb);
        }
      } else if (cnt[L * 4 + 3] > 0) {
        const double tb = sum[L * 4 + 3] / cnt[L * 4 + 3];
        c.t_bwd_ns = (int64_t)std::llround(tb);
        c.t_fwd_ns = (int64_t)std::llround(tb / 3.0);  // logits GEMM = 1 of its 3 GEMMs
      }
      out[l] = c;
    }
  });
}

// Per-launch records of the profiled steps (same clock as rp_timeline).
RP_API int rp_runtime_profile_records(rp_runtime_t* p, rp_prof_record_t* out, int64_t cap,
                                      int64_t* n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    rt->sync_all();
    *n = (int64_t)rt->prof.size();
    if (*n > cap) throw RtError(RP_E_TOOSMALL, "profile record capacity");
    std::vector<cudaEvent_t> anchor(rt->ndev, nullptr);
    for (auto& G : rt->gpus)
      if (!anchor[G.dev]) anchor[G.dev] = G.anchor;
    for (int64_t i = 0; i < *n; ++i) {
      const auto& r = rt->prof[(std::size_t)i];
      const int dev = rt->gpus[r.worker].dev;
      float a = 0.f, b = 0.f;
      RP_CUDA(cudaEventElapsedTime(&a, anchor[dev], r.a));
      RP_CUDA(cudaEventElapsedTime(&b, anchor[dev], r.b));
      out[i] = rp_prof_record_t{r.cat, r.worker, r.lane, 0,
                                (int64_t)std::llround((double)a * 1e6),
                                (int64_t)std::llround((double)b * 1e6), r.work};
    }
  });
}

// Realised optimizer hand-off edges (RP_RT_RECORD_PROTOCOL): every
// protocol wait the controller enqueued, as (kind, group, iteration) of the
// action waited on -> of the waiting action (ActionKind numbering of
// consistency.hpp; group -1 = embedding, L = head).
RP_API int rp_runtime_protocol_edges(rp_runtime_t* p, rp_protocol_edge_rec_t* out, int64_t cap,
                                     int64_t* n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    *n = (int64_t)rt->proto.size();
    if (*n > cap) throw RtError(RP_E_TOOSMALL, "protocol edge capacity");
    for (int64_t i = 0; i < *n; ++i) {
      const auto& e = rt->proto[(std::size_t)i];
      out[i] = rp_protocol_edge_rec_t{e.bk, e.bg - 1, e.bi, e.ak, e.ag - 1, e.ai};
    }
  });
}

// Host-side view of the flag words (no synchronisation): the latest
// ParamCopy index published for a group (-1: none since creation / load) and
// the latest iteration whose loss is on the host.
RP_API int rp_runtime_progress(rp_runtime_t* p, int32_t group, int32_t* published,
                               int32_t* loss_iteration) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    const int g = gidx(rt, group);
    if (published) *published = (int32_t)rt->flags.read(rt->flag_pub(g)) - 1;
    if (loss_iteration) {
      uint32_t m = 0;
      for (int w = 0; w < rt->N; ++w) m = std::max(m, rt->flags.read(rt->flag_loss(w)));
      *loss_iteration = (int32_t)m - 1;
    }
  });
}

// Measured transfer / optimizer intervals: kind 0 weight upload, 1 p_copy,
// 2 AdamW over one group (first H2D .. last D2H). Same clock as rp_timeline.
RP_API int rp_transfer_timeline(rp_runtime_t* p, rp_xfer_event_t* out, int64_t cap, int64_t* n) {
  return rt_guard([&] {
    Runtime* rt = R(p);
    rt->sync_all();
    *n = (int64_t)rt->xfers.size();
    if (*n > cap) throw RtError(RP_E_TOOSMALL, "transfer timeline capacity");
    std::vector<cudaEvent_t> anchor(rt->ndev, nullptr);
    for (auto& G : rt->gpus)
      if (!anchor[G.dev]) anchor[G.dev] = G.anchor;
    for (int64_t i = 0; i < *n; ++i) {
      const auto& r = rt->xfers[(std::size_t)i];
      float a = 0.f, b = 0.f;
      const int dev = rt->gpus[r.worker].dev;
      RP_CUDA(cudaEventElapsedTime(&a, anchor[dev], r.a));
      RP_CUDA(cudaEventElapsedTime(&b, anchor[dev], r.b));
      out[i] = rp_xfer_event_t{r.kind, r.group, r.iteration, r.worker,
                               (int64_t)std::llround((double)a * 1e6),
                               (int64_t)std::llround((double)b * 1e6)};
    }
  });
}
