/* roundpipe-b200 runtime C-ABI: the B200 executor of the RoundPipe step.
 *
 * Mirrors the paper's runtime interface:
 *   rp_forward_backward()  — micro-batches the step, plans (reference
 *       partitioner + dispatcher, cached), walks the dispatch list on the
 *       GPUs and returns as soon as the loss is known (early return);
 *   rp_step()              — queues the optimizer (fused AdamW on streamed
 *       fp32 state chunks, written back to pinned host memory); returns
 *       immediately. Sync mode applies it before the next iteration's
 *       uploads, async mode is the staleness-1 hand-off of the paper;
 *   rp_sync()              — drains everything.
 * Host buffers are plain pointers; no torch types cross this ABI.
 */
#ifndef RP_RUNTIME_H_
#define RP_RUNTIME_H_
#include <stdint.h>

#include "rp/cabi.h"
#include "rp/kernels.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rp_runtime rp_runtime_t;

enum {
  RP_RT_SKIP_INIT = 1,       /* do not randomise weights (caller loads them) */
  RP_RT_RECORD_TIMELINE = 2, /* record per-task CUDA events (measured bubble) */
  /* whole model in one fused slot (N <= 2): the forward + LM head of
   * micro-batch k+1 runs on a second stream beside k's backward (two
   * activation sets; measured no faster at the 1 kW power cap) */
  RP_RT_FUSED_PIPELINE = 4,
  /* SwiGLU as separate kernels instead of the gate/up and down GEMM
   * epilogues (the path T < 256 always takes; kept selectable for tests) */
  RP_RT_UNFUSED_SWIGLU = 8,
  /* record the (action, group, iteration) wait edges of the optimizer
   * hand-off protocol the runtime realises (rp_runtime_protocol_edges) */
  RP_RT_RECORD_PROTOCOL = 16,
  /* one worker: publish every AdamW result through the pinned bf16 master
   * (p_copy, then upload) as with several workers, instead of writing the
   * HBM-resident groups' new weights in place (keeps the host master current) */
  RP_RT_HOST_PUBLISH = 32,
  /* N > 1: each worker allocates weights / grads / AdamW output / checkpoints
   * on demand from a per-worker pool and returns them after their last use
   * (its footprint is its working set, not the model). Automatic when one
   * buffer per group and worker would not fit in HBM. */
  RP_RT_POOLED = 64
};

typedef struct {
  const char* model;           /* configs/models name or JSON path */
  int32_t seq_len;             /* s */
  int32_t micro_batch;         /* b: sequences per micro-batch */
  int32_t micro_batches;       /* M per iteration */
  int32_t round_micro_batches; /* M_R; 0 = M (single round per iteration) */
  int32_t num_gpus;            /* N devices (0..N-1) driven by this process */
  int32_t async_optimizer;     /* 1 = RoundPipe (staleness-1), 0 = RoundPipe-sync */
  int64_t mem_limit_bytes;     /* partitioner memory limit; 0 = 90% of HBM */
  double residency_factor;     /* partitioner residency (reference default 2.0) */
  const rp_layer_cost_t* costs;/* optional cost table, L+1 rows (NULL = cost model) */
  int32_t n_costs;
  rp_adam_hparams_t adam;
  uint64_t init_seed;
  float init_std;
  int32_t flags;               /* RP_RT_* */
  /* LoRA: rank r > 0 freezes every base weight
   * (embedding, norms, linears, LM head) and trains rank-r adapters on the
   * four linears of each layer: Y = X W^T + (alpha/r) (X A^T) B^T. Base
   * weights still stream from pinned host memory; grads and AdamW state exist
   * only for the adapters. 0 = full fine-tune. */
  int32_t lora_rank;
  float lora_alpha;
  /* fp32 AdamW state placement (single device): < 0 keeps the state of the
   * largest groups that fit in free HBM resident (the rest streams), 0 keeps
   * ALL of it in pinned host memory, streamed through the GPU every step
   * (BASELINE configs[2], host-offloaded Adam), > 0 caps the resident state
   * at that many GB. A zero-initialised config is host-offloaded. */
  double resident_state_gb;
  /* rows of the LM-head logits chunk [rows, V] (multiple of 128; 0 = 2048) */
  int32_t logits_rows;
  int32_t reserved_;
} rp_runtime_config_t;

typedef struct {
  int32_t num_layers;          /* L decoder layers; pseudo-layer L is the head */
  int32_t num_slots;           /* S of the plan */
  int64_t params_total;
  int64_t host_bytes_pinned;
  /* device allocations by category, all workers: 0 weights (bf16, both
   * versions), 1 fp32 grads, 2 pending AdamW output, 3 activations, 4
   * scratch, 5 checkpoints + hand-offs, 6 optimizer chunk ring, 7
   * HBM-resident fp32 AdamW state; pooled slabs count under their use */
  int64_t device_bytes[8];
  int64_t h2d_bytes, d2h_bytes, p2p_bytes; /* cumulative */
  int32_t iterations_done;
  int32_t kernels_launched;    /* cumulative count of this library's kernel launches */
  int32_t pad_;
  int64_t resident_params;     /* params whose fp32 AdamW state lives in HBM (1 device) */
  int64_t pool_peak_bytes;     /* pooled workers: max over workers of the peak bytes in use */
  int64_t pool_bytes;          /* pooled workers: slab bytes allocated, all workers */
} rp_runtime_stats_t;

int rp_runtime_create(const rp_runtime_config_t* cfg, rp_runtime_t** out);
int rp_runtime_destroy(rp_runtime_t* rt);

/* The stage plan and per-slot durations the executor runs. */
int rp_runtime_plan(rp_runtime_t* rt, rp_stage_plan_t* plan, int64_t* slot_durs,
                    int32_t cap, int32_t* n_slots);

/* Parameter groups: -1 = embedding, 0..L-1 decoder layers, L = head.
 * Values are fp32 in the flat order of include/rp/layout. */
int rp_param_count(rp_runtime_t* rt, int32_t group, int64_t* n);
int rp_set_params(rp_runtime_t* rt, int32_t group, const float* values, int64_t n);
/* which: 0 fp32 master, 1 bf16 master (as fp32), 2 last iteration's grads,
 *        3 Adam m, 4 Adam v */
int rp_get_params(rp_runtime_t* rt, int32_t group, int32_t which, float* out, int64_t n);

/* tokens/labels: host int32 [M, b, s]; labels < 0 are ignored. *loss = mean
 * token cross-entropy of the step (returned as soon as it is known). */
/* Host-state checkpoint / resume: fp32 master, Adam m/v,
 * step counters and the bf16 master of every group, plus which groups hold
 * an unpublished (staleness-1) AdamW result. Drains the runtime first. */
int rp_runtime_save(rp_runtime_t* rt, const char* path);
int rp_runtime_load(rp_runtime_t* rt, const char* path);

int rp_forward_backward(rp_runtime_t* rt, const int32_t* tokens, const int32_t* labels,
                        float* loss);
/* Non-blocking form: enqueue the iteration on every worker and return at
 * once (*iteration = its index); rp_loss() waits for the loss of one of the
 * two most recent iterations. With S=1 plans on N>1 GPUs this lets iteration
 * t+1 run on the next GPU while t finishes (the blocking call serialises
 * them, since S=1's loss is known only at the end). */
int rp_forward_backward_async(rp_runtime_t* rt, const int32_t* tokens, const int32_t* labels,
                              int32_t* iteration);
int rp_loss(rp_runtime_t* rt, int32_t iteration, float* loss);
int rp_step(rp_runtime_t* rt);
int rp_sync(rp_runtime_t* rt);

/* Measured per-task compute intervals (ns on a common clock), emission
 * order of the dispatch list; feed to rp_interior_bubble / rp_idle_in_window. */
int rp_timeline(rp_runtime_t* rt, rp_timed_event_t* out, int64_t cap, int64_t* n);
int rp_runtime_stats(rp_runtime_t* rt, rp_runtime_stats_t* stats);
int rp_timeline_clear(rp_runtime_t* rt);
/* Measured transfer / optimizer intervals (same clock as rp_timeline):
 * kind 0 = weight upload of a group, 1 = p_copy, 2 = AdamW over a group. */
typedef struct {
  int32_t kind, group, iteration, worker;
  int64_t start_ns, end_ns;
} rp_xfer_event_t;
int rp_transfer_timeline(rp_runtime_t* rt, rp_xfer_event_t* out, int64_t cap, int64_t* n);
/* The cost table the plan was built from (L+1 rows). */
int rp_runtime_costs(rp_runtime_t* rt, rp_layer_cost_t* out, int32_t cap, int32_t* n);
/* Flat layout of a group: (offset, rows, cols) per tensor, order
 * embedding: [table]; layer: in_norm qkv q_norm k_norm o post_norm gate_up down
 * (+ LoRA: qkv_A qkv_B o_A o_B gate_up_A gate_up_B down_A down_B);
 * head: final_norm lm_head. */
int rp_param_layout(rp_runtime_t* rt, int32_t group, int64_t* offs, int64_t* rows,
                    int64_t* cols, int32_t cap, int32_t* n);
const char* rp_runtime_last_error(void);
/* Kernel profiling of the following steps (CUDA events around each launch on
 * its own stream). Read: per category 0 GEMM (FLOPs), 1 attention (FLOPs),
 * 2 HBM-bound stage kernels (bytes), 3 AdamW (bytes): summed kernel ms,
 * algorithmic work and launch count. */
int rp_runtime_profile(rp_runtime_t* rt, int32_t enable);
int rp_runtime_profile_read(rp_runtime_t* rt, double* time_ms, double* work, int64_t* launches);
/* Per-launch records of the profiled steps (same clock as rp_timeline):
 * category as above, worker, lane (0 compute stream, 1 optimizer stream). */
typedef struct {
  int32_t cat, worker, lane, pad;
  int64_t start_ns, end_ns;
  double work;
} rp_prof_record_t;
/* Measured cost table (L+1 rows) from the profiled steps: per layer the mean
 * kernel ns of one micro-batch's forward (t_fwd) and forward+backward
 * (t_bwd); bytes from the cost model. Feed back as rp_runtime_config_t.costs
 * (or to rp_partition) to re-plan on measured costs. */
/* Realised optimizer hand-off edges (needs RP_RT_RECORD_PROTOCOL): every
 * protocol wait the controller enqueued — (kind, group, iteration) of the
 * action waited on -> of the waiting action; kinds as consistency.hpp
 * ActionKind (0 param upload, 1 grad write, 2 opt step, 3 p_copy, 4
 * g_copy); group -1 = embedding, 0..L-1 layers, L = head. Compare with
 * rp_build_protocol(L+1, T, event-per-layer) (tests/test_protocol_gpu.py). */
typedef struct {
  int32_t before_kind, before_group, before_iteration;
  int32_t after_kind, after_group, after_iteration;
} rp_protocol_edge_rec_t;
int rp_runtime_protocol_edges(rp_runtime_t* rt, rp_protocol_edge_rec_t* out, int64_t cap,
                              int64_t* n);
/* Host-mapped flag words, read without synchronising: the latest p_copy
 * (ParamCopy index) published for `group` (-1 none) and the latest iteration
 * whose loss is on the host. */
int rp_runtime_progress(rp_runtime_t* rt, int32_t group, int32_t* published,
                        int32_t* loss_iteration);
int rp_runtime_measured_costs(rp_runtime_t* rt, rp_layer_cost_t* out, int32_t cap, int32_t* n);
int rp_runtime_profile_records(rp_runtime_t* rt, rp_prof_record_t* out, int64_t cap, int64_t* n);

/* Device-memory plan of a configuration for one worker, computed on the
 * host without a GPU: the activation-aware stage plan the runtime would use
 * (mem_limit_bytes = 90 % of hbm_bytes minus the fixed per-worker buffers
 * unless cfg->mem_limit_bytes is set), the fixed buffers, the bytes of one
 * buffer per parameter group (2 weight versions, 2 grad buffers, AdamW
 * output, checkpoints), and for pooled workers the peak of the worst worker
 * replayed over the dispatch list. pooled = 1 if the runtime would pool. */
typedef struct {
  int32_t num_slots, pooled;
  int32_t pool_worker, pad_;
  int64_t mem_limit_bytes;
  int64_t activations, scratch, handoff, optimizer_ring, workspace;
  int64_t static_groups;
  int64_t pool_peak, pool_weights, pool_grads, pool_pend, pool_checkpoints;
  int64_t total_static, total_pooled;
} rp_memory_plan_t;
int rp_memory_plan(const rp_runtime_config_t* cfg, int64_t hbm_bytes, rp_memory_plan_t* out);

#ifdef __cplusplus
}
#endif
#endif /* RP_RUNTIME_H_ */
