/* roundpipe-b200 kernel C-ABI: the sm_100a kernels of one RoundPipe stage.
 * Device pointers + a cudaStream_t passed as void*; return codes as in
 * include/rp/cabi.h. Callable from the C++ runtime and, for tests, through
 * ctypes with torch-allocated buffers. Layouts are row-major; "ld" is the
 * row pitch in elements.
 */
#ifndef RP_KERNELS_H_
#define RP_KERNELS_H_
#include <stdint.h>
#include "rp/cabi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* D[M,N] (+)= A[M,K] . B[N,K]^T  (bf16 in, fp32 accumulate in TMEM).
 * a_mn_major=0: A stored [M,K] (lda >= K);  1: A stored [K,M] (lda >= M).
 * b_mn_major=0: B stored [N,K] (ldb >= K);  1: B stored [K,N] (ldb >= N).
 * out_f32=0: D bf16 = acc (+ R, a bf16 [M,N] residual, optional);
 * out_f32=1: D fp32 = acc, or D += acc when accumulate=1. */
typedef struct {
  int32_t M, N, K;
  const void* A; int64_t lda; int32_t a_mn_major;
  const void* B; int64_t ldb; int32_t b_mn_major;
  void* D; int64_t ldd; int32_t out_f32; int32_t accumulate;
  const void* R; int64_t ldr;
} rp_gemm_args_t;
int rp_gemm_bf16(const rp_gemm_args_t* args, void* stream);
/* Why the last rp_gemm_* call of this thread failed ("" after a success):
 * the precondition, tensor-map encode or launch step that refused it. */
const char* rp_gemm_last_error(void);
/* D = A . B^T + A2 . B2^T (+ R / accumulate as in rp_gemm_bf16): a second K
 * segment of K2 columns with the same majors as A and B (A2 [M,K2] or [K2,M],
 * B2 [N,K2] or [K2,N]). Used for LoRA: X W^T + U B^T and dY W + dU A in one
 * GEMM. */
int rp_gemm_bf16_2seg(const rp_gemm_args_t* args, const void* A2, int64_t lda2, const void* B2,
                      int64_t ldb2, int32_t K2, void* stream);
/* Down-projection dgrad fused with the SwiGLU backward: acc = A . B^T is
 * dact [M,N] (A [M,K] K-major, B [K,N] MN-major); R = gu = [g | u] [M,2N]
 * (pitch ldr), D = dgu = [dg | du] [M,2N] bf16 (pitch ldd); dact is never
 * stored. Equals rp_gemm_bf16 into a bf16 dact followed by rp_swiglu_bwd.
 * N % 8 == 0, out_f32 = accumulate = 0. */
int rp_gemm_swiglu_bwd(const rp_gemm_args_t* args, void* stream);
/* Gate/up projection fused with the SwiGLU forward: B = W_gu [2N, K]
 * (K-major, gate rows then up rows), A [M, K] K-major; D = gu = [g | u]
 * [M, 2N] bf16 (kept for the backward) and act = silu(g) * u [M, N] bf16
 * (pitch ld_act). args->N is N (half of W_gu's rows); R unused. Equals
 * rp_gemm_bf16 into gu followed by rp_swiglu_fwd. N % 8 == 0. */
int rp_gemm_swiglu_fwd(const rp_gemm_args_t* args, void* act, int64_t ld_act, void* stream);
/* Every GEMM epilogue with an optional second K segment: epilogue 0 =
 * rp_gemm_bf16, 1 = rp_gemm_swiglu_bwd, 2 = rp_gemm_swiglu_fwd (act, ld_act);
 * K2 > 0 adds A2 . B2^T as rp_gemm_bf16_2seg does (for the SwiGLU epilogues
 * M >= 256). LoRA runs its gate/up and down linears through this. */
int rp_gemm_ex(const rp_gemm_args_t* args, int32_t epilogue, void* act, int64_t ld_act,
               const void* A2, int64_t lda2, const void* B2, int64_t ldb2, int32_t K2,
               void* stream);

/* AdamW hyper-parameters (decoupled weight decay), fp32. */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay, grad_scale;
} rp_adam_hparams_t;

/* RMSNorm over rows of h (h % 8 == 0): y = bf16(w * x * rstd). */
int rp_rmsnorm_fwd(const void* x, int64_t ldx, const void* w, void* y, int64_t ldy,
                   float* rstd, int32_t rows, int32_t h, float eps, void* stream);
/* dx = rstd*(dy*w - xhat*mean(dy*w*xhat)) [+ dres]; dx32 (fp32) and/or dx16
 * (bf16) outputs; dw[h] += sum_rows dy*xhat (fp32, atomics). Rows dense.
 * dy | x | dres rows are staged through a bulk-copy ring when h >= 1024,
 * rows % 4 == 0 and dy, x, rstd, dres are 16-byte aligned; otherwise a
 * register version runs (same math; fp32 contraction may differ in the last
 * bit). */
int rp_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd,
                   const float* dres, float* dx32, void* dx16, float* dw, int32_t rows,
                   int32_t h, void* stream);
/* Per-head RMSNorm of q and k slots of the fused qkv row + RoPE (rotate_half,
 * cos_sin = float2 (cos, sin) table [seq, head_dim/2]); position = t % seq.
 * head_dim 64 or 128, T % 128 == 0, ld % 8 == 0; every pointer 16-byte
 * aligned (operands are staged by 1-D bulk copies) -> RP_E_INPUT otherwise.
 * The backward bulk-copies rstd when nq % 4 == 0 and nk % 4 == 0 and reads
 * it from global memory otherwise. */
int rp_qk_norm_rope_fwd(const void* qkv, int64_t ld, int32_t nq, int32_t nk,
                        int32_t head_dim, const void* qw, const void* kw,
                        const float* cos_sin, int32_t seq, void* q_out, void* k_out,
                        float* rstd_q, float* rstd_k, int32_t T, float eps, void* stream);
int rp_qk_norm_rope_bwd(const void* dq, const void* dk, const void* qkv, int64_t ld,
                        int32_t nq, int32_t nk, int32_t head_dim, const void* qw,
                        const void* kw, const float* rstd_q, const float* rstd_k,
                        const float* cos_sin, int32_t seq, void* dqkv, int64_t ldd,
                        float* dqw, float* dkw, int32_t T, void* stream);
/* gu rows = [gate | up] (2m); act = silu(gate) * up. */
int rp_swiglu_fwd(const void* gu, void* act, int64_t T, int32_t m, void* stream);
int rp_swiglu_bwd(const void* dact, const void* gu, void* dgu, int64_t T, int32_t m,
                  void* stream);
/* out[t] = table[ids[t]] (table: device or host-mapped pinned memory). */
int rp_embed_fwd(const int32_t* ids, const void* table, void* out, int32_t T, int32_t h,
                 void* stream);
/* dE[ids[t]] += dx[t] (fp32). */
int rp_embed_bwd(const int32_t* ids, const float* dx, float* dE, int32_t T, int32_t h,
                 void* stream);
/* Cross-entropy over a bf16 logits chunk [rows, V]: loss_sum += lse - z[label]
 * (label < 0 ignored), logits overwritten IN PLACE by (softmax - onehot) *
 * grad_scale; row_lse optional. */
int rp_ce_fwd_bwd(void* logits, int64_t ld, const int32_t* labels, int32_t rows, int32_t V,
                  float grad_scale, float* loss_sum, float* row_lse, void* stream);
/* AdamW on one fp32 state chunk (in place); w16 (optional) receives bf16
 * weights. step >= 1 is the bias-correction step. */
int rp_adamw(float* master, float* m, float* v, const float* grad, void* w16, int64_t n,
             const rp_adam_hparams_t* hp, int32_t step, void* stream);
int rp_f32_to_bf16(const float* a, void* b, int64_t n, void* stream);
int rp_bf16_to_f32(const void* a, float* b, int64_t n, void* stream);
int rp_add_f32(float* a, const float* b, int64_t n, void* stream);
/* a[i] *= f (bf16 in place; LoRA scaling of the rank-r projections) */
int rp_scale_bf16(void* a, int64_t n, float f, void* stream);
/* Deterministic N(0, std) rounded to bf16 (counter hash + Box-Muller); f32
 * (optional) receives the exact widening of the bf16 value. */
int rp_init_normal(float* f32, void* b16, int64_t n, uint64_t seed, float std, void* stream);
int rp_fill(float* f32, void* b16, int64_t n, float value, void* stream);

/* Causal GQA flash attention forward on the 5th-gen tensor cores (tcgen05 +
 * TMEM + TMA), head_dim 64 or 128, bf16 in/out.
 * q [T, nq, hd] (row pitch ldq), k/v [T, nk, hd] (pitch ldk/ldv), o [T, nq, hd];
 * lse [nq, T] fp32 (natural log). Sequences are packed: T = batch * seq and
 * attention never crosses a seq boundary. 16-byte aligned base pointers and
 * pitches. */
int rp_attn_fwd_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                   int64_t ldv, void* o, int64_t ldo, float* lse, int32_t T, int32_t seq,
                   int32_t nq, int32_t nk, int32_t head_dim, float scale, void* stream);
/* Backward on the 5th-gen tensor cores; dq/dk/dv bf16 with the layouts of
 * q/k/v (own pitches). head_dim 128 with an even GQA group: one key-major
 * kernel per (key block, query-head pair) forms dK, dV and dQ (dQ^T = K^T
 * dS^T reduce-added into a per-stream fp32 accumulator in L2). Otherwise a
 * dK/dV kernel plus a query-major dQ kernel that recomputes S and dP. GQA
 * partials of dK/dV are summed in fp32. Workspaces: delta fp32 [nq, T];
 * dkv_acc fp32 [2, T, nk*head_dim]. */
int rp_attn_bwd_tc(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                   int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                   const float* lse, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                   int64_t lddv, float* delta, float* dkv_acc, int32_t T, int32_t seq,
                   int32_t nq, int32_t nk, int32_t head_dim, float scale, void* stream);

/* ---- mixture of experts (Qwen3-MoE; csrc/kernels/moe.cu) ----------------
 * Grouped GEMM: rows [row_off[e], row_off[e+1]) of A (K-major, args->M rows
 * in all) and D times expert e's B, the e-th block of b_group_rows rows of B
 * (K-major [groups*N, K]: b_group_rows = N; MN-major [groups*K, N]:
 * b_group_rows = K). row_off: DEVICE int32[groups+1]. epilogue 0: bf16 D
 * (+ R); 1: SwiGLU backward (R = gu, D = dgu, B MN-major). */
int rp_gemm_grouped(const rp_gemm_args_t* args, const int32_t* row_off, int32_t groups,
                    int32_t b_group_rows, int32_t epilogue, void* stream);
/* softmax (fp32) over E router logits [T, E] -> top-k experts and weights
 * (renormalised over the k when norm_topk), per-expert counts [E] (zeroed
 * here). E <= 256, k <= 32. */
int rp_moe_route(const float* logits, int32_t T, int32_t E, int32_t k, int32_t norm_topk,
                 int32_t* topk_idx, float* topk_w, int32_t* counts, void* stream);
/* counts -> offsets [E+1] (cursor [E] scratch); row pos[t*k+j] of the
 * expert-sorted buffers for every (token, slot); xs[pos] = x[t] [.., h],
 * w_s[pos] = topk_w[t, j] */
int rp_moe_permute(const void* x, int64_t ldx, int32_t T, int32_t h, int32_t k, int32_t E,
                   const int32_t* topk_idx, const float* topk_w, const int32_t* counts,
                   int32_t* offsets, int32_t* cursor, int32_t* pos, float* w_s, void* xs,
                   void* stream);
/* xs[pos[t*k+j]] = x[t] */
int rp_moe_gather(const void* x, int64_t ldx, int32_t T, int32_t h, int32_t k,
                  const int32_t* pos, void* xs, void* stream);
/* out[t] = res[t] (optional) + sum_j topk_w[t,j] ys[pos[t*k+j]]  (fp32 sum, bf16 out) */
int rp_moe_combine(const void* ys, const int32_t* pos, const float* topk_w, int32_t T,
                   int32_t k, int32_t h, const void* res, int64_t ldr, void* out, int64_t ldo,
                   void* stream);
/* dh[t] = dh32[t] + sum_j dxs[pos[t*k+j]]  (dh32 fp32 [T, h], dh bf16) */
int rp_moe_combine_bwd(const void* dxs, const int32_t* pos, int32_t T, int32_t k, int32_t h,
                       const float* dh32, void* dh, int64_t ldd, void* stream);
/* per expert-sorted row r: dw_s[r] = <dact[r], silu(g) u>, dgu[r] =
 * swiglu'(w_s[r] dact[r]) with gu = [g | u] [rows, 2m] */
int rp_moe_swiglu_bwd(const void* dact, const void* gu, const float* w_s, int64_t rows,
                      int32_t m, void* dgu, float* dw_s, void* stream);
/* d(router logits) [T, E] (bf16) from dw through the top-k renormalisation and
 * the softmax */
int rp_moe_router_bwd(const float* logits, int32_t T, int32_t E, int32_t k, int32_t norm_topk,
                      const int32_t* topk_idx, const int32_t* pos, const float* dw_s,
                      void* dlogits, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RP_KERNELS_H_ */
