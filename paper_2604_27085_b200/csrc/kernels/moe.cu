// Mixture-of-experts routing / permutation kernels (sm_100a) for Qwen3-MoE
// decoder layers (BASELINE configs[4], Qwen3-235B-A22B; router restated from
// transformers 5.5.0 modeling_qwen3_moe.py:254-272, experts :215-251).
//
// Forward of one MoE MLP over T tokens, k of E experts per token:
//   logits = h2 . Wg^T                       (router GEMM, fp32 out)
//   rp_moe_route     softmax (fp32) -> top-k -> (optionally) renormalised
//                    weights; per-expert token counts
//   rp_moe_permute   counts -> row offsets (exclusive scan); every (token,
//                    slot) gets a row of the expert-sorted buffers; gathers
//                    the token's input row there (and its weight)
//   grouped GEMMs    gu_s = x_s W_gu[e]^T, act_s = silu(g) u, y_s = act_s W_d[e]^T
//                    (rp_gemm_grouped: rows of expert e x its weights)
//   rp_moe_combine   out[t] = res[t] + sum_j w[t,j] y_s[pos[t,j]]   (fp32 sum)
// Backward (experts and router frozen, as in the LoRA fine-tune of C5; the
// gradient still flows through both into the layer input):
//   rp_moe_gather    dy_s[pos] = dY[t]                   (unweighted)
//   grouped GEMM     dact'_s = dy_s W_d[e]
//   rp_moe_swiglu_bwd  dw_s = <dact'_s, act_s>, dgu_s = swiglu'(w_s dact'_s)
//   grouped GEMM     dx_s = dgu_s W_gu[e]
//   rp_moe_router_bwd  dlogits from dw through the renormalisation and softmax
//   router dgrad GEMM  dh32 = dlogits . Wg
//   rp_moe_combine_bwd dh[t] = dh32[t] + sum_j dx_s[pos[t,j]]   (bf16 out)
// Rows of one expert are in an arbitrary (atomics) order; every row is
// computed independently and every per-token sum runs over j = 0..k-1 in
// order, so results do not depend on it.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels/swiglu.cuh"
#include "rp/kernels.h"

namespace rp {
namespace {

typedef __nv_bfloat16 bf16;
constexpr int MAXE = 256, MAXK = 32;

int status() { return cudaGetLastError() == cudaSuccess ? RP_OK : RP_E_CUDA; }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one warp per token; lane l holds experts l, l+32, ... (E <= 256)
__global__ void moe_route_kernel(const float* __restrict__ logits, int T, int E, int k, int norm,
                                 int32_t* __restrict__ idx, float* __restrict__ w,
                                 int32_t* __restrict__ counts) {
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (t >= T) return;
  const float* row = logits + (long long)t * E;
  float p[MAXE / 32];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) {
    const int e = lane + 32 * i;
    p[i] = e < E ? row[e] : -INFINITY;
    mx = fmaxf(mx, p[i]);
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) {
    p[i] = lane + 32 * i < E ? expf(p[i] - mx) : 0.f;
    sum += p[i];
  }
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) p[i] *= inv;
  // top-k by repeated warp argmax (ties -> lower expert index)
  float my_v = 0.f, tot = 0.f;  // lane j keeps the j-th selection
  int my_e = 0;
  for (int j = 0; j < k; ++j) {
    float bv = -1.f;
    int be = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < MAXE / 32; ++i) {
      const int e = lane + 32 * i;
      if (e < E && (p[i] > bv || (p[i] == bv && e < be))) {
        bv = p[i];
        be = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      if (ov > bv || (ov == bv && oe < be)) {
        bv = ov;
        be = oe;
      }
    }
    if (lane == j) {
      my_v = bv;
      my_e = be;
    }
    tot += bv;
#pragma unroll
    for (int i = 0; i < MAXE / 32; ++i)
      if (lane + 32 * i == be) p[i] = -2.f;  // taken
  }
  if (lane < k) {
    idx[(long long)t * k + lane] = my_e;
    w[(long long)t * k + lane] = norm ? my_v / tot : my_v;
    atomicAdd(&counts[my_e], 1);
  }
}

// single block: exclusive scan of the counts -> offsets[E+1]; cursors reset
__global__ void moe_offsets_kernel(const int32_t* __restrict__ counts, int E,
                                   int32_t* __restrict__ off, int32_t* __restrict__ cursor) {
  __shared__ int s[MAXE + 1];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      s[e] = acc;
      acc += counts[e];
    }
    s[E] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= E; e += blockDim.x) {
    off[e] = s[e];
    if (e < E) cursor[e] = 0;
  }
}

// one warp per token: rows for its k slots, gather x[t] into them (16 B lanes)
__global__ void moe_permute_kernel(const bf16* __restrict__ x, long long ldx, int T, int h, int k,
                                   const int32_t* __restrict__ idx, const float* __restrict__ w,
                                   const int32_t* __restrict__ off, int32_t* __restrict__ cursor,
                                   int32_t* __restrict__ pos, float* __restrict__ w_s,
                                   bf16* __restrict__ xs) {
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (t >= T) return;
  int my = 0;
  if (lane < k) {
    const int e = idx[(long long)t * k + lane];
    my = off[e] + atomicAdd(&cursor[e], 1);
    pos[(long long)t * k + lane] = my;
    w_s[my] = w[(long long)t * k + lane];
  }
  const uint4* src = reinterpret_cast<const uint4*>(x + (long long)t * ldx);
  for (int j = 0; j < k; ++j) {
    const int r = __shfl_sync(0xffffffffu, my, j);
    uint4* dst = reinterpret_cast<uint4*>(xs + (long long)r * h);
    for (int c = lane; c < h / 8; c += 32) dst[c] = src[c];
  }
}

// dy_s[pos[t, j]] = dy[t] for every slot j (one warp per token)
__global__ void moe_gather_kernel(const bf16* __restrict__ x, long long ldx, int T, int h, int k,
                                  const int32_t* __restrict__ pos, bf16* __restrict__ xs) {
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (t >= T) return;
  const uint4* src = reinterpret_cast<const uint4*>(x + (long long)t * ldx);
  for (int j = 0; j < k; ++j) {
    uint4* dst = reinterpret_cast<uint4*>(xs + (long long)pos[(long long)t * k + j] * h);
    for (int c = lane; c < h / 8; c += 32) dst[c] = src[c];
  }
}

__device__ __forceinline__ void ld8(const bf16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const bf16* b = reinterpret_cast<const bf16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(b[i]);
}
__device__ __forceinline__ void st8(bf16* p, const float (&f)[8]) {
  uint4 u;
  bf16* b = reinterpret_cast<bf16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = __float2bfloat16_rn(f[i]);
  *reinterpret_cast<uint4*>(p) = u;
}

// out[t] = res[t] + sum_j w[t,j] ys[pos[t,j]]  (block per token, fp32 sum)
__global__ void moe_combine_kernel(const bf16* __restrict__ ys, const int32_t* __restrict__ pos,
                                   const float* __restrict__ w, int k, int h,
                                   const bf16* __restrict__ res, long long ldr,
                                   bf16* __restrict__ out, long long ldo) {
  const long long t = blockIdx.x;
  for (int c = threadIdx.x * 8; c < h; c += blockDim.x * 8) {
    float acc[8];
    if (res) {
      ld8(res + t * ldr + c, acc);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    }
    float part[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < k; ++j) {
      float y[8];
      ld8(ys + (long long)pos[t * k + j] * h + c, y);
      const float wj = w[t * k + j];
#pragma unroll
      for (int i = 0; i < 8; ++i) part[i] = fmaf(wj, y[i], part[i]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += part[i];
    st8(out + t * ldo + c, acc);
  }
}

// dh[t] = dh32[t] + sum_j dxs[pos[t,j]]  (bf16 out)
__global__ void moe_combine_bwd_kernel(const bf16* __restrict__ dxs, const int32_t* __restrict__ pos,
                                       int k, int h, const float* __restrict__ dh32,
                                       bf16* __restrict__ dh, long long ldd) {
  const long long t = blockIdx.x;
  for (int c = threadIdx.x * 8; c < h; c += blockDim.x * 8) {
    float acc[8];
    const float4 a = *reinterpret_cast<const float4*>(dh32 + t * h + c);
    const float4 b = *reinterpret_cast<const float4*>(dh32 + t * h + c + 4);
    float part[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < k; ++j) {
      float y[8];
      ld8(dxs + (long long)pos[t * k + j] * h + c, y);
#pragma unroll
      for (int i = 0; i < 8; ++i) part[i] += y[i];
    }
    acc[0] = a.x + part[0];
    acc[1] = a.y + part[1];
    acc[2] = a.z + part[2];
    acc[3] = a.w + part[3];
    acc[4] = b.x + part[4];
    acc[5] = b.y + part[5];
    acc[6] = b.z + part[6];
    acc[7] = b.w + part[7];
    st8(dh + t * ldd + c, acc);
  }
}

// per expert-sorted row r: act = silu(g) u (bf16, as the forward's down GEMM
// read it), dw_s[r] = <dact'_r, act_r>, dgu = swiglu'(w_s[r] dact'_r)
__global__ void __launch_bounds__(256) moe_swiglu_bwd_kernel(const bf16* __restrict__ dact,
                                                             const bf16* __restrict__ gu,
                                                             const float* __restrict__ w_s, int m,
                                                             bf16* __restrict__ dgu,
                                                             float* __restrict__ dw_s) {
  const long long r = blockIdx.x;
  const bf16* g_row = gu + r * 2 * m;
  const bf16* a_row = dact + r * m;
  bf16* d_row = dgu + r * 2 * m;
  const float wr = w_s[r];
  float dot = 0.f;
  for (int c = threadIdx.x * 8; c < m; c += 256 * 8) {
    float d[8], g[8], u[8], dg[8], du[8];
    ld8(a_row + c, d);
    ld8(g_row + c, g);
    ld8(g_row + m + c, u);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float act = __bfloat162float(__float2bfloat16_rn(swiglu_fwd_elem(g[i], u[i])));
      dot = fmaf(d[i], act, dot);
      swiglu_bwd_elem(wr * d[i], g[i], u[i], dg[i], du[i]);
    }
    st8(d_row + c, dg);
    st8(d_row + m + c, du);
  }
  __shared__ float red[8];
  dot = warp_sum(dot);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += red[i];
    dw_s[r] = s;
  }
}

// d(router logits) of one token (warp): q = softmax(logits); selected set S,
// Z = sum_S q; w_j = q_j / Z (norm) or q_j. dq_i = (dw_i - sum_j dw_j w_j) / Z
// on S (norm) or dw_i; dlogit_e = q_e (dq_e - sum_i q_i dq_i). bf16 out (the
// A operand of the router dgrad GEMM).
__global__ void moe_router_bwd_kernel(const float* __restrict__ logits, int T, int E, int k,
                                      int norm, const int32_t* __restrict__ idx,
                                      const int32_t* __restrict__ pos,
                                      const float* __restrict__ dw_s, bf16* __restrict__ dlogits) {
  const int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (t >= T) return;
  const float* row = logits + (long long)t * E;
  float q[MAXE / 32];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) {
    const int e = lane + 32 * i;
    q[i] = e < E ? row[e] : -INFINITY;
    mx = fmaxf(mx, q[i]);
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) {
    q[i] = lane + 32 * i < E ? expf(q[i] - mx) : 0.f;
    sum += q[i];
  }
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) q[i] *= inv;
  // the k selected experts: (expert, q, dw) broadcast from lanes 0..k-1
  int my_e = 0;
  float my_dw = 0.f;
  if (lane < k) {
    my_e = idx[(long long)t * k + lane];
    my_dw = dw_s[pos[(long long)t * k + lane]];
  }
  float Z = 0.f, swd = 0.f;
  for (int j = 0; j < k; ++j) {
    const int e = __shfl_sync(0xffffffffu, my_e, j);
    const float dwj = __shfl_sync(0xffffffffu, my_dw, j);
    float qe = 0.f;
#pragma unroll
    for (int i = 0; i < MAXE / 32; ++i)
      if (lane + 32 * i == e) qe = q[i];
    qe = warp_sum(qe);
    Z += qe;
    swd += dwj * qe;
  }
  // dq on the selected experts; sum_i q_i dq_i
  float dq[MAXE / 32];
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) dq[i] = 0.f;
  for (int j = 0; j < k; ++j) {
    const int e = __shfl_sync(0xffffffffu, my_e, j);
    const float dwj = __shfl_sync(0xffffffffu, my_dw, j);
    const float v = norm ? (dwj - swd / Z) / Z : dwj;
#pragma unroll
    for (int i = 0; i < MAXE / 32; ++i)
      if (lane + 32 * i == e) dq[i] = v;
  }
  float qdq = 0.f;
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) qdq += q[i] * dq[i];
  qdq = warp_sum(qdq);
#pragma unroll
  for (int i = 0; i < MAXE / 32; ++i) {
    const int e = lane + 32 * i;
    if (e < E) dlogits[(long long)t * E + e] = __float2bfloat16_rn(q[i] * (dq[i] - qdq));
  }
}

}  // namespace
}  // namespace rp

using namespace rp;
#define RP_API extern "C" __attribute__((visibility("default")))

RP_API int rp_moe_route(const float* logits, int32_t T, int32_t E, int32_t k, int32_t norm_topk,
                        int32_t* topk_idx, float* topk_w, int32_t* counts, void* stream) {
  if (T < 0 || E <= 0 || E > MAXE || k <= 0 || k > MAXK || k > E || k > 32) return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  if (cudaMemsetAsync(counts, 0, sizeof(int32_t) * E, s) != cudaSuccess) return RP_E_CUDA;
  if (T == 0) return RP_OK;
  moe_route_kernel<<<(T + 7) / 8, 256, 0, s>>>(logits, T, E, k, norm_topk, topk_idx, topk_w, counts);
  return status();
}

RP_API int rp_moe_permute(const void* x, int64_t ldx, int32_t T, int32_t h, int32_t k, int32_t E,
                          const int32_t* topk_idx, const float* topk_w, const int32_t* counts,
                          int32_t* offsets, int32_t* cursor, int32_t* pos, float* w_s, void* xs,
                          void* stream) {
  if (T < 0 || h % 8 || ldx % 8 || E <= 0 || E > MAXE || k <= 0 || k > 32) return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  moe_offsets_kernel<<<1, 256, 0, s>>>(counts, E, offsets, cursor);
  if (T > 0)
    moe_permute_kernel<<<(T + 7) / 8, 256, 0, s>>>((const bf16*)x, ldx, T, h, k, topk_idx, topk_w,
                                                  offsets, cursor, pos, w_s, (bf16*)xs);
  return status();
}

RP_API int rp_moe_gather(const void* x, int64_t ldx, int32_t T, int32_t h, int32_t k,
                         const int32_t* pos, void* xs, void* stream) {
  if (T < 0 || h % 8 || ldx % 8 || k <= 0) return RP_E_INPUT;
  if (T == 0) return RP_OK;
  moe_gather_kernel<<<(T + 7) / 8, 256, 0, (cudaStream_t)stream>>>((const bf16*)x, ldx, T, h, k,
                                                                  pos, (bf16*)xs);
  return status();
}

RP_API int rp_moe_combine(const void* ys, const int32_t* pos, const float* topk_w, int32_t T,
                          int32_t k, int32_t h, const void* res, int64_t ldr, void* out,
                          int64_t ldo, void* stream) {
  if (T < 0 || h % 8 || ldo % 8 || (res && ldr % 8) || k <= 0) return RP_E_INPUT;
  if (T == 0) return RP_OK;
  moe_combine_kernel<<<T, 128, 0, (cudaStream_t)stream>>>((const bf16*)ys, pos, topk_w, k, h,
                                                         (const bf16*)res, ldr, (bf16*)out, ldo);
  return status();
}

RP_API int rp_moe_combine_bwd(const void* dxs, const int32_t* pos, int32_t T, int32_t k, int32_t h,
                              const float* dh32, void* dh, int64_t ldd, void* stream) {
  if (T < 0 || h % 8 || ldd % 8 || k <= 0) return RP_E_INPUT;
  if (T == 0) return RP_OK;
  moe_combine_bwd_kernel<<<T, 128, 0, (cudaStream_t)stream>>>((const bf16*)dxs, pos, k, h, dh32,
                                                             (bf16*)dh, ldd);
  return status();
}

RP_API int rp_moe_swiglu_bwd(const void* dact, const void* gu, const float* w_s, int64_t rows,
                             int32_t m, void* dgu, float* dw_s, void* stream) {
  if (m % 8 || rows < 0) return RP_E_INPUT;
  if (rows == 0) return RP_OK;
  moe_swiglu_bwd_kernel<<<(unsigned)rows, 256, 0, (cudaStream_t)stream>>>(
      (const bf16*)dact, (const bf16*)gu, w_s, m, (bf16*)dgu, dw_s);
  return status();
}

RP_API int rp_moe_router_bwd(const float* logits, int32_t T, int32_t E, int32_t k, int32_t norm_topk,
                             const int32_t* topk_idx, const int32_t* pos, const float* dw_s,
                             void* dlogits, void* stream) {
  if (T < 0 || E <= 0 || E > MAXE || k <= 0 || k > 32 || k > E) return RP_E_INPUT;
  if (T == 0) return RP_OK;
  moe_router_bwd_kernel<<<(T + 7) / 8, 256, 0, (cudaStream_t)stream>>>(
      logits, T, E, k, norm_topk, topk_idx, pos, dw_s, (bf16*)dlogits);
  return status();
}
