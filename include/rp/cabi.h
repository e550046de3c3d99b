/* roundpipe-b200 C ABI.
 *
 * One shared library (paper_2604_27085_b200/libroundpipe_b200.so) exports:
 *   1. planning — the reference planner API (proj/include/roundpipe headers)
 *      behind plain C: cost table, partition, dispatch list, expected
 *      timeline/bubble, LPT transfer windows, consistency protocol;
 *   2. kernels  — the sm_100a compute kernels of one RoundPipe stage
 *      (device pointers + cudaStream_t, see include/rp/kernels.h);
 *   3. runtime  — the B200 executor that walks the dispatch list
 *      (see include/rp/runtime.h).
 *
 * Conventions (reference error taxonomy: proj/tools/roundpipe.cpp:25-29):
 *   return 0 ok, 2 bad input, 3 infeasible, 4 protocol violation,
 *   5 cap exceeded / internal, 6 CUDA error, 7 output buffer too small.
 *   No C++ exception crosses the ABI; rp_last_error() returns the message of
 *   the last failing call on the calling thread. Variable-length outputs are
 *   caller-owned arrays with an explicit capacity; the required count is
 *   always written to *n, so a call with cap 0 is a size query.
 */
#ifndef RP_CABI_H_
#define RP_CABI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  RP_OK = 0,
  RP_E_INPUT = 2,
  RP_E_INFEASIBLE = 3,
  RP_E_VIOLATION = 4,
  RP_E_INTERNAL = 5,
  RP_E_CUDA = 6,
  RP_E_TOOSMALL = 7
};

/* ScheduleKind (reference: scheduler.hpp:19-26) */
enum {
  RP_SCHED_ROUNDPIPE = 0,
  RP_SCHED_ROUNDPIPE_SYNC = 1,
  RP_SCHED_GPIPE = 2,
  RP_SCHED_1F1B = 3,
  RP_SCHED_INTERLEAVED_1F1B = 4,
  RP_SCHED_LOOPED_BFS = 5
};
/* ProtocolMode (reference: consistency.hpp:28) */
enum { RP_PROTO_BLOCKING = 0, RP_PROTO_EVENT_PER_MODEL = 1, RP_PROTO_EVENT_PER_LAYER = 2 };
/* ActionKind (reference: consistency.hpp:27) */
enum { RP_ACT_PARAM_UPLOAD = 0, RP_ACT_GRAD_WRITE = 1, RP_ACT_OPT_STEP = 2,
       RP_ACT_PARAM_COPY = 3, RP_ACT_GRAD_COPY = 4 };
/* StageKind (reference: partitioner.hpp:32) */
enum { RP_STAGE_FWD = 0, RP_STAGE_BWD = 1, RP_STAGE_FUSED = 2 };

/* POD mirrors of the reference value types */
typedef struct { /* ModelConfig, cost_model.hpp:16-42 */
  double hidden_dim;
  int32_t num_heads, num_kv_heads;
  double intermediate_dim;
  int32_t active_experts, total_experts, num_layers;
  int32_t has_head; /* head_flops_per_token present */
  double head_flops_per_token;
  int32_t has_head_param_bytes;
  double head_param_bytes;
} rp_model_config_t;

typedef struct { /* GpuSpec, cost_model.hpp:44-56 */
  double peak_fp16_flops, memory_bytes, link_bandwidth;
} rp_gpu_spec_t;

typedef struct { /* LayerCost, cost_model.hpp:70-76 */
  int64_t t_fwd_ns, t_bwd_ns, param_bytes, act_ckpt_bytes, act_full_bytes;
} rp_layer_cost_t;

typedef struct { int32_t first, last; } rp_layer_range_t; /* LayerRange */

typedef struct { /* StagePlan, partitioner.hpp:34-44; fwd/bwd caller-owned */
  int32_t num_fwd, num_bwd; /* bwd excludes the fused stage */
  rp_layer_range_t fused;
  int64_t t_max_ns, objective;
  rp_layer_range_t* fwd;
  rp_layer_range_t* bwd;
  int32_t cap; /* capacity of fwd and of bwd (L always suffices) */
} rp_stage_plan_t;

typedef struct { /* Task, scheduler.hpp:61-68 */
  int32_t iteration, round, slot, mb, gpu, pad_;
  int64_t dur_ns;
} rp_task_t;

typedef struct { /* TimedEvent, simulator.hpp:17-21 */
  rp_task_t task;
  int64_t start_ns, end_ns;
} rp_timed_event_t;

typedef struct { /* SimReport scalars, simulator.hpp:34-44 */
  int64_t makespan_ns, span_ns, busy_total_ns, bubble_num, bubble_den;
  double bubble_ratio;
} rp_sim_report_t;

typedef struct { /* one LPT chunk placement, transfer_planner.hpp:23-39 */
  int32_t item;        /* index into the caller's item list */
  int32_t chunk_index;
  int32_t window;
  int32_t position;    /* order inside its window */
  int64_t bytes;
} rp_transfer_chunk_t;

typedef struct { /* WindowVerdict, transfer_planner.hpp:144-150 */
  int32_t slot, feasible;
  int64_t window_ns, weight_bytes, activation_bytes;
} rp_window_verdict_t;

typedef struct { int32_t kind, layer, iteration; } rp_protocol_action_t;
typedef struct { int32_t before, after; } rp_protocol_edge_t;

typedef struct { /* ActionDurations, consistency.hpp:257-274 */
  int64_t upload_ns, grad_write_ns, step_ns, p_copy_ns, g_copy_ns;
} rp_action_durations_t;

const char* rp_last_error(void);
const char* rp_version(void);

/* ---- planning (reentrant) ---------------------------------------------- */

/* cost_model::layer_costs (cost_model.hpp:185) */
int rp_layer_costs(const rp_model_config_t* cfg, int32_t seq_len,
                   int32_t micro_batch, const rp_gpu_spec_t* gpu,
                   int32_t include_head, rp_layer_cost_t* out, int32_t cap,
                   int32_t* n);

/* config_io::load_model / load_gpu (config_io.hpp:50,73) */
int rp_load_model(const char* name_or_path, rp_model_config_t* out);
int rp_load_gpu(const char* name_or_path, rp_gpu_spec_t* out);

/* partitioner::candidate_tmax (partitioner.hpp:84) */
int rp_candidate_tmax(const rp_layer_cost_t* costs, int32_t L, int64_t* out,
                      int64_t cap, int64_t* n);

/* partitioner::optimal_partition (partitioner.hpp:199) */
int rp_partition(const rp_layer_cost_t* costs, int32_t L, int32_t num_gpus,
                 int32_t micro_batches, int64_t mem_limit_bytes,
                 double residency_factor, rp_stage_plan_t* plan);

/* partitioner::greedy_pack at one t_max; *found = 0 when it returns nullopt */
int rp_greedy_pack(const rp_layer_cost_t* costs, int32_t L, int32_t num_gpus,
                   int32_t micro_batches, int64_t mem_limit_bytes,
                   double residency_factor, int64_t t_max,
                   rp_stage_plan_t* plan, int32_t* found);

/* partitioner::symmetric_split (partitioner.hpp:220) */
int rp_symmetric_split(const rp_layer_cost_t* costs, int32_t L,
                       int32_t num_stages, rp_layer_range_t* out, int32_t cap,
                       int32_t* n);

/* scheduler::slot_table_from_plan durations (scheduler.hpp:104) */
int rp_slot_durations(const rp_stage_plan_t* plan, const rp_layer_cost_t* costs,
                      int32_t L, int64_t* out, int32_t cap, int32_t* n);

/* scheduler::synthesize (scheduler.hpp:236). Round-robin kinds read
 * slot_durs[0..S); baselines read stage_fwd/bwd_durs[0..n_stages). */
int rp_synthesize(int32_t kind, int32_t num_gpus, int32_t micro_batches,
                  int32_t round_micro_batches, int32_t iterations,
                  const int64_t* slot_durs, int32_t S,
                  const int64_t* stage_fwd_durs, const int64_t* stage_bwd_durs,
                  int32_t n_stages, rp_task_t* out, int64_t cap, int64_t* n,
                  int32_t* num_gpus_out, int32_t* slots_per_iteration);

/* scheduler::default_round_micro_batches (scheduler.hpp:97) */
int32_t rp_default_round_micro_batches(int32_t M, int32_t N);

/* scheduler::validate (scheduler.hpp:255): RP_OK or RP_E_INPUT + message */
int rp_validate_schedule(int32_t kind, int32_t num_gpus,
                         int32_t slots_per_iteration, const rp_task_t* tasks,
                         int64_t n);

/* simulator::simulate (simulator.hpp:48); events[] has n entries */
int rp_simulate(int32_t kind, int32_t num_gpus, int32_t slots_per_iteration,
                const rp_task_t* tasks, int64_t n, int32_t barrier,
                int64_t optimizer_delay_ns, rp_sim_report_t* report,
                int64_t* busy_per_gpu, rp_timed_event_t* events);

/* simulator::idle_in_window / interior_bubble (simulator.hpp:153,172),
 * applied to any timeline (simulated or measured) */
int rp_idle_in_window(const rp_timed_event_t* events, int64_t n,
                      int32_t num_gpus, int64_t w0, int64_t w1, int64_t* num,
                      int64_t* den, double* ratio);
int rp_interior_bubble(const rp_timed_event_t* events, int64_t n,
                       int32_t num_gpus, int32_t iter_lo, int32_t iter_hi,
                       int64_t* num, int64_t* den, double* ratio);

/* transfer_planner::plan (transfer_planner.hpp:73). ids[i] are the tensor ids
 * (ordering key), out[] lists chunks window by window in placement order. */
/* svg::render_gantt (svg.hpp:26) of a simulated or measured timeline;
 * slot_kinds: 0 fwd, 1 fused, 2 bwd (optional legend). NUL-terminated SVG
 * into out; cap 0 = size query, *len = length without the NUL. */
int rp_render_gantt(const rp_timed_event_t* events, int64_t n, int32_t num_gpus,
                    const int32_t* slot_kinds, const rp_layer_range_t* slot_layers,
                    int32_t n_slots, int32_t width, char* out, int64_t cap, int64_t* len);

/* SimReport scalars (simulator.hpp:134-151) over a measured timeline. */
int rp_timeline_report(const rp_timed_event_t* events, int64_t n, int32_t num_gpus,
                       rp_sim_report_t* report, int64_t* busy_per_gpu);

int rp_transfer_plan(const char* const* ids, const int64_t* bytes,
                     const int32_t* directions, int32_t n_items,
                     int32_t num_windows, int64_t max_chunk_bytes,
                     rp_transfer_chunk_t* out, int64_t cap, int64_t* n,
                     int64_t* window_totals, int64_t* makespan_bytes);

/* transfer_planner::optimal_makespan (transfer_planner.hpp:104) */
int rp_optimal_makespan(const int64_t* chunks, int32_t n, int32_t num_windows,
                        int64_t* makespan);

/* transfer_planner::stage_feasibility (transfer_planner.hpp:158) */
int rp_stage_feasibility(const rp_stage_plan_t* plan,
                         const rp_layer_cost_t* costs, int32_t L,
                         const rp_gpu_spec_t* gpu, int32_t micro_batches,
                         rp_window_verdict_t* out, int32_t cap, int32_t* n);

/* consistency::build_protocol (consistency.hpp:84) */
int rp_build_protocol(int32_t layers, int32_t iterations, int32_t mode,
                      int32_t drop_edge, rp_protocol_action_t* actions,
                      int64_t action_cap, int64_t* n_actions,
                      int32_t* gpu_actions, rp_protocol_edge_t* edges,
                      int64_t edge_cap, int64_t* n_edges);

/* consistency::check_all_interleavings (consistency.hpp:172) on the built
 * protocol; returns RP_OK with *ok=1, or RP_E_VIOLATION with the violated
 * constraint and witness, or RP_E_INTERNAL when the state cap is hit. */
int rp_check_protocol(int32_t layers, int32_t iterations, int32_t mode,
                      int32_t drop_edge, int64_t max_states, int32_t* ok,
                      int32_t* violated, rp_protocol_action_t* witness,
                      int64_t cap, int64_t* n);

/* consistency::protocol_makespan (consistency.hpp:279) */
int rp_protocol_makespan(int32_t layers, int32_t iterations, int32_t mode,
                         int32_t drop_edge, const rp_action_durations_t* dur,
                         int64_t* makespan);

#ifdef __cplusplus
}
#endif

#endif /* RP_CABI_H_ */
