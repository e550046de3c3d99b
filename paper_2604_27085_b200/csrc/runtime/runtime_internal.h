// Internal structures of the roundpipe-b200 executor (see runtime.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <array>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "roundpipe/roundpipe.hpp"
#include "rp/kernels.h"
#include "rp/runtime.h"

namespace rp {
namespace rt {

struct RtError : std::runtime_error {
  int code;
  RtError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define RP_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::rp::rt::RtError(RP_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_) + \
                                             " @" + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)
#define RP_K(expr)                                                                     \
  do {                                                                                 \
    int c_ = (expr);                                                                   \
    if (c_ != RP_OK)                                                                   \
      throw ::rp::rt::RtError(c_, std::string("kernel failed: ") + #expr + " -> " +    \
                                      cudaGetErrorString(cudaGetLastError()));          \
  } while (0)

// Decoder shape (Qwen3 family).
struct Shape {
  int h = 0, nq = 0, nk = 0, hd = 0, m = 0, L = 0, V = 0;
  // mixture of experts (Qwen3-MoE): E experts of intermediate size m, ek
  // routed per token, top-k weights renormalised when norm_topk
  int E = 1, ek = 1;
  bool norm_topk = true;
  bool moe() const { return E > 1; }
  double theta = 1e6, eps = 1e-6;
  int qd() const { return nq * hd; }
  int kd() const { return nk * hd; }
  int qkvd() const { return qd() + 2 * kd(); }
};

// Flat parameter layout of one group; every tensor starts on a 128-element
// (256-byte) boundary so TMA/vector loads are aligned.
struct Tensor {
  int64_t off = 0, rows = 0, cols = 1;
  int64_t numel() const { return rows * cols; }
};
struct LayerLayout {
  // dense: gate_up [2m x h], down [h x m]; MoE: router [E x h], gate_up
  // [E*2m x h] (per expert gate rows then up rows), down [E*h x m]
  Tensor in_norm, qkv, q_norm, k_norm, o, post_norm, router, gate_up, down;
  // LoRA adapters (rank r > 0), after the base tensors: A [r x in], B [out x r]
  // (MoE layers: attention projections only — experts and router frozen)
  Tensor qkv_A, qkv_B, o_A, o_B, gu_A, gu_B, down_A, down_B;
  int64_t lora_off = 0;  // start of the adapters (= total without LoRA)
  int64_t total = 0;
};
struct HeadLayout {
  Tensor final_norm, lm_head;
  int64_t total = 0;
};
LayerLayout make_layer_layout(const Shape& s, int lora_rank = 0);
HeadLayout make_head_layout(const Shape& s);

// Pinned host state of one parameter group: fp32 optimizer copy (master,
// m, v) and the bf16 master copy the GPUs upload.
struct HostGroup {
  int64_t n = 0;
  // trainable region [t_off, n): 0 for full fine-tune; the adapters' offset in
  // LoRA mode; n for a frozen group. master/m/v (and device grads / resident
  // state) exist only for it — the pointers are shifted so that global
  // offsets index them (valid for offsets >= t_off).
  int64_t t_off = 0;
  int64_t tn() const { return n - t_off; }
  uint16_t* w16 = nullptr;
  float* master = nullptr;
  float* m = nullptr;
  float* v = nullptr;
  int step = 0;
  // single-device runs keep the fp32 state of some groups resident in free
  // HBM (device 0): AdamW then runs without the PCIe round trip; the host
  // copy is refreshed on demand (read_state / save) and re-uploaded on writes
  float* d_state = nullptr;  // [master | m | v], 3n fp32, or null (streamed)
  bool host_stale = false;   // host master/m/v older than d_state
  // single worker (N = 1): a resident group's AdamW writes its bf16 output
  // straight into the device weight buffer of the iteration that will use it
  // (no pend buffer, no p_copy / upload round trip over PCIe); the host bf16
  // master is then refreshed on demand
  bool direct = false;
  bool w16_stale = false;
};

// Device-side state of one parameter group on one worker.
struct DevGroup {
  uint16_t* w[2] = {nullptr, nullptr};    // bf16 weights, by iteration parity: the
                                          // upload of t+1 streams in under t's compute
  int loaded[2] = {-1, -1};               // iteration whose version each buffer holds
  float* grad[2] = {nullptr, nullptr};    // fp32 accumulators by iteration parity
  uint16_t* pend = nullptr;               // AdamW output awaiting p_copy
  cudaEvent_t ev_upload[2] = {nullptr, nullptr};   // upload(l, t) into w[t%2]   GPU lane
  cudaEvent_t ev_lastuse[2] = {nullptr, nullptr};  // last compute read of w[b] (WAR)
  cudaEvent_t ev_gradwrite = nullptr;     // GradWrite(l, t)           GPU lane
  cudaEvent_t ev_adam[2] = {nullptr, nullptr};  // g_copy: AdamW consumed grad[p]
  int adam_iter[2] = {-1, -1};            // iteration whose grads that AdamW consumed
  cudaEvent_t ev_pcopy = nullptr;         // p_copy(l, t)              optimizer lane
  cudaEvent_t ev_state = nullptr;         // fp32 state written back to host
  bool up_started = false;                // windowed upload: first chunk enqueued
  cudaEvent_t up_xa = nullptr;            // its transfer-timeline start event
  // pooled workers (N > 1): the buffers above are slabs of the worker's pool,
  // bound for one version / iteration and returned after their last use
  int w_slab[2] = {-1, -1}, grad_slab[2] = {-1, -1}, pend_slab = -1;
};

// A device buffer of a worker's pool (exact-size classes). It is handed out
// by the controller; its next user's stream waits on free_ev, recorded where
// the previous user's last access was enqueued. `tag_*` names the action
// that last released it (for the realised-protocol record).
struct Slab {
  void* p = nullptr;
  std::size_t bytes = 0;
  cudaEvent_t free_ev = nullptr;
  bool recorded = false, busy = false;
  int cat = 0;
  int tag_kind = -1, tag_group = -1, tag_iter = -1;
};

// Activations of one decoder layer for one micro-batch.
struct LayerActs {
  uint16_t *x, *h1, *qkv, *q, *k, *o, *x2, *h2, *gu, *act;
  float *rstd1, *rstd_q, *rstd_k, *lse, *rstd2;
  uint16_t *u_qkv = nullptr, *u_o = nullptr, *u_gu = nullptr, *u_down = nullptr;  // LoRA: s X A^T
  // MoE: router logits [T, E] (fp32), top-k experts / weights / expert-sorted
  // rows [T, ek], routing weight per sorted row, expert row offsets [E+1];
  // gu / act then hold the T*ek expert-sorted rows
  float* r_logits = nullptr;
  int32_t *r_idx = nullptr, *r_pos = nullptr, *r_off = nullptr;
  float *r_w = nullptr, *r_ws = nullptr;
  const uint16_t* xin = nullptr;  // the input actually used by layer_fwd
  cudaEvent_t ev_free = nullptr;        // weight-gradient GEMMs done reading act/h2/o/h1
  cudaEvent_t ev_chain_free = nullptr;  // the dgrad chain done with this layer's activations
};

// A hand-off / checkpoint buffer with its producer and consumer events. The
// producer records `ready` on ITS stream after the write; cudaEventRecord
// needs an event of the stream's device, and the producer of a checkpoint
// buffer changes with the round, so there is one ready event per producer
// device (created there on first use). The consumer (this buffer's device)
// records `read` after its last read; cross-device waits on either are legal.
struct Slotbuf {
  void* p = nullptr;
  int slab = -1;                       // pooled checkpoints: slab of the consumer's pool
  std::vector<cudaEvent_t> ready_dev;  // by producer device
  cudaEvent_t ready = nullptr;         // the one last recorded (what consumers wait on)
  cudaEvent_t read = nullptr;
};

// One logical RoundPipe worker ("stateless GPU"). Workers map onto physical
// devices (worker % device_count); N workers on one B200 exercise the full
// N-way dispatch in tests.
struct Gpu {
  int id = 0, dev = 0;
  cudaStream_t compute = nullptr, act = nullptr, w_h2d = nullptr;
  cudaStream_t opt_h2d = nullptr, opt_d2h = nullptr, opt_comp = nullptr;
  cudaStream_t opt_res = nullptr;  // AdamW of HBM-resident groups (never queued behind PCIe)
  // weight-gradient GEMMs run here, off the dgrad chain on `compute`, so the
  // persistent GEMMs' partial last waves and the chain's HBM-bound kernels
  // overlap them; scratch gradients they read are double-buffered
  cudaStream_t wgrad = nullptr;
  uint16_t* dx16s[2] = {nullptr, nullptr};
  uint16_t* dgus[3] = {nullptr, nullptr, nullptr};  // ring: the fused down-dgrad
  static constexpr int n_dgu = 3;                     // writes dgu one GEMM earlier
  int dgu_i = 0;
  uint16_t* dqkvs[2] = {nullptr, nullptr};
  cudaEvent_t ev_dx16_free[2] = {nullptr, nullptr};
  cudaEvent_t ev_dgu_free[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_dqkv_free[2] = {nullptr, nullptr};
  cudaEvent_t ev_wgrad = nullptr;  // last weight-gradient GEMM enqueued
  int bwd_par = 0;
  // cross-stream fork events, reused round-robin (a wait captures the event's
  // state when it is enqueued, so re-recording an old one is safe)
  cudaEvent_t fork_ev[64] = {};
  int fork_i = 0;
  std::vector<DevGroup> groups;           // index g = group + 1 (0 = embedding)
  std::vector<LayerActs> acts;            // per decoder layer of the fused stage
  // pipelined fused stage (whole model fused, N <= 2): the forward + LM head of
  // micro-batch k+1 runs on `fwd2` while micro-batch k's backward runs on
  // `compute`; micro-batches alternate between two activation sets
  std::vector<LayerActs> acts2;
  cudaStream_t fwd2 = nullptr;
  float* hdx32 = nullptr;                 // head output gradient, handed to the backward
  uint16_t *hdx16 = nullptr, *hdh = nullptr;
  cudaEvent_t ev_head_done = nullptr, ev_hdx_free = nullptr, ev_fwd_join = nullptr;
  float* dx32[2] = {nullptr, nullptr};
  uint16_t *dx16 = nullptr, *dh = nullptr, *dact = nullptr, *dgu = nullptr, *dattn = nullptr;
  uint16_t *dqkv = nullptr, *dq_t = nullptr, *dk_t = nullptr;
  uint16_t* du = nullptr;  // LoRA: s dY B of the linear being back-propagated (T x r)
  // MoE scratch: expert-sorted rows (gathered inputs / dY, expert outputs /
  // input grads), counts and cursors, dact', dL/dw per row, router grads
  uint16_t *m_xs = nullptr, *m_ys = nullptr, *m_dact = nullptr, *m_dlogits = nullptr;
  int32_t *m_counts = nullptr, *m_cursor = nullptr;
  float *m_dws = nullptr, *m_dh32 = nullptr;
  float *dq_acc = nullptr, *delta = nullptr;
  uint16_t* xbuf[2] = {nullptr, nullptr};
  uint16_t *hN = nullptr, *logits = nullptr;
  float *rstdN = nullptr, *loss_dev = nullptr;
  int32_t *tokens_dev = nullptr, *labels_dev = nullptr;  // current iteration's parity set
  // per iteration parity: token/label/loss buffers, so iteration t+1 can be
  // enqueued (non-blocking forward_backward) while t still runs
  int32_t *tokens_par[2] = {nullptr, nullptr}, *labels_par[2] = {nullptr, nullptr};
  float* loss_par[2] = {nullptr, nullptr};
  cudaEvent_t ev_iter_done[2] = {nullptr, nullptr};  // last read of parity set (compute)
  cudaEvent_t ev_loss_par[2] = {nullptr, nullptr};
  float* cos_sin = nullptr;
  // streamed-AdamW chunk ring: kOptSlots x (master, m, v) chunks (3 slots
  // measured 2-4 % slower than 2 on the C3 headline, profiles/r02q_ab.jsonl:
  // more DMA in flight delays the weight uploads sharing the H2D lane)
  static constexpr int kOptSlots = 2;
  float* opt_buf[kOptSlots][3] = {};
  cudaEvent_t opt_free[kOptSlots] = {};
  int opt_slot = 0;
  // hand-offs by round parity and micro-batch: activations (bf16) into a
  // forward/fused slot, gradients (fp32) into a backward slot
  std::vector<Slotbuf> hand_act, hand_grad;   // [parity * MR + mb]
  std::vector<Slotbuf> ckpt;                  // [(parity * L + l) * MR + mb]
  cudaEvent_t anchor = nullptr;
  cudaEvent_t ev_tokens = nullptr;
  std::vector<std::size_t> allocated;
  std::vector<void*> owned;  // every device allocation of this worker (freed by ~Runtime)
  std::vector<Slab> slabs;   // pooled buffers (weights, grads, AdamW output, checkpoints)
  std::size_t pool_bytes = 0, pool_busy = 0, pool_peak = 0;
};

// ---- memory plan (memory_plan.cpp) ------------------------------------------------
// Per-worker device bytes that do not scale with the parameter groups.
struct WorkerBytes {
  int64_t activations = 0, scratch = 0, handoff = 0, optimizer_ring = 0, workspace = 0;
  int64_t fixed() const;
};
WorkerBytes worker_fixed_bytes(const Shape& s, int T, int seq, int M, int MR, int S, int parities,
                               int nsets, int logits_rows, int lora_r, int64_t chunk_elems);
// Peak of a pooled worker's group buffers (the worst worker), by category.
struct PoolPeak {
  int worker = 0;
  int64_t total = 0, weights = 0, grads = 0, pend = 0, checkpoints = 0;
};
PoolPeak pooled_peak(const Shape& s, const LayerLayout& LL, const HeadLayout& HL,
                     const roundpipe::StagePlan& plan,
                     const std::vector<roundpipe::StageSlot>& slots,
                     const roundpipe::Schedule& sched, int N, int MR, int T, bool async,
                     int lora_r, int iters);
// The stage plan of a configuration: the reference partitioner on the cost
// table (cfg.costs or the cost model), given cfg.mem_limit_bytes, or else
// 90 % of the device's HBM minus what a worker holds besides parameters
// (activation-aware, iterated until the fused stage's activation sets fit).
struct PlanChoice {
  std::vector<roundpipe::LayerCost> costs;
  roundpipe::StagePlan plan;
  std::vector<roundpipe::StageSlot> slots;
  int64_t mem_limit = 0;
  WorkerBytes fixed;
};
Shape load_shape(const std::string& model);
PlanChoice choose_plan(const rp_runtime_config_t& cfg, const Shape& s, const std::string& model,
                       int64_t hbm_bytes, int logits_rows, int64_t chunk_elems);

struct TaskRecord {
  roundpipe::Task task;
  int worker;
  cudaEvent_t start, end;
};

}  // namespace rt
}  // namespace rp
