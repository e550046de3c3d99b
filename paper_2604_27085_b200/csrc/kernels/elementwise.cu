// HBM-bound kernels of one Qwen3 decoder stage (sm_100a):
//   RMSNorm fwd/bwd, fused per-head QK-RMSNorm + RoPE fwd/bwd, SwiGLU fwd/bwd,
//   embedding gather / scatter-add, LM-head cross-entropy (in-place dlogits),
//   fused AdamW on a streamed fp32 state chunk, and small utilities.
// All are 16-byte vectorised, fp32 internally; reductions of parameter grads
// go registers -> shared memory -> one atomicAdd per column per block.
// Math follows transformers' Qwen3 (modeling_qwen3.py: RMSNorm :50-67,
// rotate_half / apply_rotary_pos_emb :151-182, MLP :70-83) in fp32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels/swiglu.cuh"
#include "rp/kernels.h"

namespace rp {
namespace {

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = bf2f(b[i]);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 u;
  __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = f2bf(f[i]);
  *reinterpret_cast<uint4*>(p) = u;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int THREADS>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < THREADS / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------- RMSNorm
// y = bf16(w * x * rstd), rstd = 1/sqrt(mean(x^2) + eps). One 128-thread
// block per row, the row held in registers (VPT 16-byte vectors per thread),
// so x is read once; many rows in flight per SM.

template <int NW>
__device__ __forceinline__ float rn_block_sum(float v, float* red) {
  v = warp_sum(v);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NW; ++i) t += red[i];
  return t;
}

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = bf2f(b[i]);
}

template <int RN_THREADS, int VPT>
__global__ void __launch_bounds__(RN_THREADS)
    rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x, long long ldx,
                       const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ y,
                       long long ldy, float* __restrict__ rstd, int h, float eps) {
  __shared__ float red[RN_THREADS / 32];
  const long long row = blockIdx.x;
  const __nv_bfloat16* xr = x + row * ldx;
  uint4 xv[VPT];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int c = (threadIdx.x + j * RN_THREADS) * 8;
    xv[j] = c < h ? *reinterpret_cast<const uint4*>(xr + c) : make_uint4(0, 0, 0, 0);
    float f[8];
    unpack8(xv[j], f);
#pragma unroll
    for (int i = 0; i < 8; ++i) ss += f[i] * f[i];
  }
  const float r = rsqrtf(rn_block_sum<RN_THREADS / 32>(ss, red) / h + eps);
  if (threadIdx.x == 0 && rstd) rstd[row] = r;
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int c = (threadIdx.x + j * RN_THREADS) * 8;
    if (c >= h) continue;
    float f[8], g[8];
    unpack8(xv[j], f);
    load8(w + c, g);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = g[i] * (f[i] * r);
    store8(y + row * ldy + c, f);
  }
}

// dx = rstd * (g - xhat * mean(g * xhat)),  g = dy * w,  xhat = x * rstd
// dx_total = dx + dres (optional fp32 residual grad); written fp32 and/or bf16.
// dw[c] += sum_rows dy * xhat. A block walks rows with a stride of gridDim.x
// (several blocks per SM keep rows in flight); dw partials stay in registers
// until one float4 atomic per 4 columns per block.
template <int RN_THREADS, int VPT>
__global__ void __launch_bounds__(RN_THREADS)
    rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                       const __nv_bfloat16* __restrict__ w, const float* __restrict__ rstd,
                       const float* __restrict__ dres, float* __restrict__ dx32,
                       __nv_bfloat16* __restrict__ dx16, float* __restrict__ dw, int rows, int h) {
  __shared__ float red[2][RN_THREADS / 32];
  uint4 wv[VPT];
  float dwa[VPT][8];
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int c = (threadIdx.x + j * RN_THREADS) * 8;
    wv[j] = c < h ? *reinterpret_cast<const uint4*>(w + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) dwa[j][i] = 0.f;
  }
  int par = 0;
  for (int row = blockIdx.x; row < rows; row += gridDim.x, par ^= 1) {
    const long long off = (long long)row * h;
    uint4 av[VPT], bv[VPT];
    float4 rv[VPT][2];  // the residual gradient, loaded with dy / x (not after the reduction)
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int c = (threadIdx.x + j * RN_THREADS) * 8;
      if (c < h) {
        av[j] = *reinterpret_cast<const uint4*>(dy + off + c);
        bv[j] = *reinterpret_cast<const uint4*>(x + off + c);
        if (dres) {
          rv[j][0] = *reinterpret_cast<const float4*>(dres + off + c);
          rv[j][1] = *reinterpret_cast<const float4*>(dres + off + c + 4);
        }
      } else {
        av[j] = bv[j] = make_uint4(0, 0, 0, 0);
      }
    }
    const float r = rstd[row];
    float dot = 0.f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      float a[8], b[8], g[8];
      unpack8(av[j], a);
      unpack8(bv[j], b);
      unpack8(wv[j], g);
#pragma unroll
      for (int i = 0; i < 8; ++i) dot += a[i] * g[i] * (b[i] * r);
    }
    dot = warp_sum(dot);
    if (threadIdx.x % 32 == 0) red[par][threadIdx.x / 32] = dot;
    __syncthreads();  // red[par] is rewritten two rows later, after another barrier
    float tot = 0.f;
#pragma unroll
    for (int i = 0; i < RN_THREADS / 32; ++i) tot += red[par][i];
    const float mean = tot / h;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int c = (threadIdx.x + j * RN_THREADS) * 8;
      if (c >= h) continue;
      float a[8], b[8], g[8], o[8];
      unpack8(av[j], a);
      unpack8(bv[j], b);
      unpack8(wv[j], g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = b[i] * r;
        o[i] = r * (a[i] * g[i] - xh * mean);
        dwa[j][i] += a[i] * xh;
      }
      if (dres) {
        const float4 d0 = rv[j][0], d1 = rv[j][1];
        o[0] += d0.x; o[1] += d0.y; o[2] += d0.z; o[3] += d0.w;
        o[4] += d1.x; o[5] += d1.y; o[6] += d1.z; o[7] += d1.w;
      }
      if (dx32) {
        *reinterpret_cast<float4*>(dx32 + off + c) = make_float4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<float4*>(dx32 + off + c + 4) = make_float4(o[4], o[5], o[6], o[7]);
      }
      if (dx16) store8(dx16 + off + c, o);
    }
  }
  if (dw && (int)blockIdx.x < rows) {
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int c = (threadIdx.x + j * RN_THREADS) * 8;
      if (c < h) {
        atomicAdd(reinterpret_cast<float4*>(dw + c),
                  make_float4(dwa[j][0], dwa[j][1], dwa[j][2], dwa[j][3]));
        atomicAdd(reinterpret_cast<float4*>(dw + c + 4),
                  make_float4(dwa[j][4], dwa[j][5], dwa[j][6], dwa[j][7]));
      }
    }
  }
}

// ------------------------------------------------------- QK-norm + RoPE
// A head of HD elements is handled by TPH = HD/8 consecutive lanes, 8
// elements (16 bytes) each; the per-head RMS reduces over those lanes and the
// rotate_half partner (element e +- HD/2) lives in lane ^ TPH/2. A 128-thread
// block covers HPB = 128/TPH heads of one token per pass and walks passes
// then tokens (grid-stride over one wave of resident blocks); a thread's
// (cos, sin) pairs depend only on its lane slot and the token, so they are
// loaded once per token. The loads of QK_NB passes are issued together
// before any of them is used (occupancy is register-limited to 5-8 blocks of
// 128 threads per SM, profiles/r02g_ncu_full.json): backward 52.2 -> 48.1 us,
// forward unchanged at 25.6 us (profiles/r02h_qk_ab.jsonl) — its remaining
// limit is the serial per-token chain (2 load rounds per token for 40 heads,
// ~5.5 tokens per block), not the loads in flight of one round.
constexpr int QK_THREADS = 128;
constexpr int QK_NB = 4;

template <int HD>
__global__ void __launch_bounds__(QK_THREADS)
    qk_norm_rope_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, long long ld, int nq, int nk,
                            const __nv_bfloat16* __restrict__ qw,
                            const __nv_bfloat16* __restrict__ kw, const float2* __restrict__ cs,
                            int seq, __nv_bfloat16* __restrict__ qo, __nv_bfloat16* __restrict__ ko,
                            float* __restrict__ rstd_q, float* __restrict__ rstd_k, int T,
                            float eps) {
  constexpr int TPH = HD / 8, HALF = HD / 2, HPB = QK_THREADS / TPH;
  const int heads = nq + nk;
  const int sub = threadIdx.x % TPH, hl = threadIdx.x / TPH;
  const bool lo = sub < TPH / 2;
  float wq[8], wk[8];
  load8(qw + sub * 8, wq);
  load8(kw + sub * 8, wk);
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const int pos = t % seq;
    const float4* c4 = reinterpret_cast<const float4*>(cs + (long long)pos * HALF + (sub * 8) % HALF);
    float4 c[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = c4[i];
    const __nv_bfloat16* row = qkv + (long long)t * ld;
    for (int base0 = 0; base0 < heads; base0 += QK_NB * HPB) {
      uint4 raw[QK_NB];
#pragma unroll
      for (int b = 0; b < QK_NB; ++b) {
        const int hh = base0 + b * HPB + hl;
        raw[b] = hh < heads ? *reinterpret_cast<const uint4*>(row + hh * HD + sub * 8)
                            : make_uint4(0, 0, 0, 0);
      }
      // every lane runs every pass (the shuffles below are warp-wide); lanes
      // whose head is past the end compute on zeros and store nothing
#pragma unroll
      for (int b = 0; b < QK_NB; ++b) {
        if (base0 + b * HPB >= heads) break;  // block-uniform
        const int hh = base0 + b * HPB + hl;
        const bool act = hh < heads;
        const bool is_q = hh < nq;
        float v[8];
        unpack8(raw[b], v);
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) ss += v[i] * v[i];
#pragma unroll
        for (int o = TPH / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        const float r = rsqrtf(ss / HD + eps);
        float n[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) n[i] = bf2f(f2bf((is_q ? wq[i] : wk[i]) * (v[i] * r)));
        float out[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float4 cc = c[i / 2];  // (cos, sin) of elements i, i+1
          const float p0 = __shfl_xor_sync(0xffffffffu, n[i], TPH / 2);
          const float p1 = __shfl_xor_sync(0xffffffffu, n[i + 1], TPH / 2);
          out[i] = lo ? n[i] * cc.x - p0 * cc.y : n[i] * cc.x + p0 * cc.y;
          out[i + 1] = lo ? n[i + 1] * cc.z - p1 * cc.w : n[i + 1] * cc.z + p1 * cc.w;
        }
        if (!act) continue;
        __nv_bfloat16* dst = is_q ? qo + ((long long)t * nq + hh) * HD
                                  : ko + ((long long)t * nk + (hh - nq)) * HD;
        store8(dst + sub * 8, out);
        if (sub == 0) {
          if (is_q) rstd_q[(long long)t * nq + hh] = r;
          else rstd_k[(long long)t * nk + (hh - nq)] = r;
        }
      }
    }
  }
}

// Backward: undo the rotation (R^T), then per-head RMSNorm backward;
// dqkv[:, q/k slots] = dx; dqw/dkw[HD] += sum(dn * xhat) (registers -> smem
// -> one atomic per column per block). Loads batched over QK_NB passes as in
// the forward.
template <int HD>
__global__ void __launch_bounds__(QK_THREADS)
    qk_norm_rope_bwd_kernel(const __nv_bfloat16* __restrict__ dq, const __nv_bfloat16* __restrict__ dk,
                            const __nv_bfloat16* __restrict__ qkv, long long ld, int nq, int nk,
                            const __nv_bfloat16* __restrict__ qw,
                            const __nv_bfloat16* __restrict__ kw, const float* __restrict__ rstd_q,
                            const float* __restrict__ rstd_k, const float2* __restrict__ cs, int seq,
                            __nv_bfloat16* __restrict__ dqkv, long long ldd, float* __restrict__ dqw,
                            float* __restrict__ dkw, int T) {
  constexpr int TPH = HD / 8, HALF = HD / 2, HPB = QK_THREADS / TPH;
  __shared__ float sq[HD], sk[HD];
  for (int i = threadIdx.x; i < HD; i += blockDim.x) sq[i] = sk[i] = 0.f;
  __syncthreads();
  const int heads = nq + nk;
  const int sub = threadIdx.x % TPH, hl = threadIdx.x / TPH;
  const bool lo = sub < TPH / 2;
  float wq[8], wk[8], aq[8], ak[8];
  load8(qw + sub * 8, wq);
  load8(kw + sub * 8, wk);
#pragma unroll
  for (int i = 0; i < 8; ++i) aq[i] = ak[i] = 0.f;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const int pos = t % seq;
    const float4* c4 = reinterpret_cast<const float4*>(cs + (long long)pos * HALF + (sub * 8) % HALF);
    float4 c[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = c4[i];
    for (int base0 = 0; base0 < heads; base0 += QK_NB * HPB) {  // warp-uniform passes (shuffles)
      uint4 graw[QK_NB], xraw[QK_NB];
      float rr[QK_NB];
#pragma unroll
      for (int b = 0; b < QK_NB; ++b) {
        const int hh = base0 + b * HPB + hl;
        graw[b] = xraw[b] = make_uint4(0, 0, 0, 0);
        rr[b] = 0.f;
        if (hh < heads) {
          const bool is_q = hh < nq;
          rr[b] = is_q ? rstd_q[(long long)t * nq + hh] : rstd_k[(long long)t * nk + (hh - nq)];
          graw[b] = *reinterpret_cast<const uint4*>(
              (is_q ? dq + ((long long)t * nq + hh) * HD : dk + ((long long)t * nk + (hh - nq)) * HD) +
              sub * 8);
          xraw[b] = *reinterpret_cast<const uint4*>(qkv + (long long)t * ld + hh * HD + sub * 8);
        }
      }
#pragma unroll
      for (int b = 0; b < QK_NB; ++b) {
        if (base0 + b * HPB >= heads) break;  // block-uniform
        const int hh = base0 + b * HPB + hl;
        const bool act = hh < heads;
        const bool is_q = hh < nq;
        const float r = rr[b];
        float gv[8], xv[8];
        unpack8(graw[b], gv);
        unpack8(xraw[b], xv);
        float dn[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float4 cc = c[i / 2];
          const float p0 = __shfl_xor_sync(0xffffffffu, gv[i], TPH / 2);
          const float p1 = __shfl_xor_sync(0xffffffffu, gv[i + 1], TPH / 2);
          dn[i] = lo ? gv[i] * cc.x + p0 * cc.y : gv[i] * cc.x - p0 * cc.y;
          dn[i + 1] = lo ? gv[i + 1] * cc.z + p1 * cc.w : gv[i + 1] * cc.z - p1 * cc.w;
        }
        float dot = 0.f, gx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          xv[i] *= r;  // xhat
          gx[i] = dn[i] * (is_q ? wq[i] : wk[i]);
          dot += gx[i] * xv[i];
          if (is_q) aq[i] += dn[i] * xv[i]; else ak[i] += dn[i] * xv[i];
        }
#pragma unroll
        for (int o = TPH / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        const float mean = dot / HD;
        float out[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) out[i] = r * (gx[i] - xv[i] * mean);
        if (act) store8(dqkv + (long long)t * ldd + hh * HD + sub * 8, out);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    atomicAdd(&sq[sub * 8 + i], aq[i]);
    atomicAdd(&sk[sub * 8 + i], ak[i]);
  }
  __syncthreads();
  if (dqw && dkw)  // null: frozen norm weights (LoRA)
    for (int i = threadIdx.x; i < HD; i += blockDim.x) {
      atomicAdd(dqw + i, sq[i]);
      atomicAdd(dkw + i, sk[i]);
    }
}

// ------------------------------------------------------------------ SwiGLU
// gu row = [gate(0..m) | up(0..m)];  act = silu(g) * u. Block-per-row (no
// integer division in the index math); 8-wide vectors.
__global__ void __launch_bounds__(256) swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu,
                                                         __nv_bfloat16* __restrict__ act, int m) {
  const long long t = blockIdx.x;
  const __nv_bfloat16* g_row = gu + t * 2 * m;
  __nv_bfloat16* a_row = act + t * m;
  for (int c = threadIdx.x * 8; c < m; c += 256 * 8) {
    float g[8], u[8], o[8];
    load8(g_row + c, g);
    load8(g_row + m + c, u);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = rp::swiglu_fwd_elem(g[k], u[k]);
    store8(a_row + c, o);
  }
}

__global__ void __launch_bounds__(256) swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ dact,
                                                         const __nv_bfloat16* __restrict__ gu,
                                                         __nv_bfloat16* __restrict__ dgu, int m) {
  const long long t = blockIdx.x;
  const __nv_bfloat16* g_row = gu + t * 2 * m;
  __nv_bfloat16* d_row = dgu + t * 2 * m;
  const __nv_bfloat16* a_row = dact + t * m;
  for (int c = threadIdx.x * 8; c < m; c += 256 * 8) {
    float d[8], g[8], u[8], dg[8], du[8];
    load8(a_row + c, d);
    load8(g_row + c, g);
    load8(g_row + m + c, u);
#pragma unroll
    for (int k = 0; k < 8; ++k) rp::swiglu_bwd_elem(d[k], g[k], u[k], dg[k], du[k]);
    store8(d_row + c, dg);
    store8(d_row + m + c, du);
  }
}

// --------------------------------------------------------------- embedding
// out[t] = table[ids[t]]; table may be device memory or host-mapped pinned
// memory (zero-copy gather over PCIe: only the T used rows cross the link).
__global__ void embed_fwd_kernel(const int32_t* __restrict__ ids,
                                 const __nv_bfloat16* __restrict__ table,
                                 __nv_bfloat16* __restrict__ out, int T, int h) {
  const int t = blockIdx.x;
  const long long row = ids[t];
  const uint4* src = reinterpret_cast<const uint4*>(table + row * h);
  uint4* dst = reinterpret_cast<uint4*>(out + (long long)t * h);
  for (int i = threadIdx.x; i < h / 8; i += blockDim.x) dst[i] = src[i];
}

// dE[ids[t]] += dx[t]  (fp32 accumulate; repeated ids handled by atomics)
__global__ void embed_bwd_kernel(const int32_t* __restrict__ ids, const float* __restrict__ dx,
                                 float* __restrict__ dE, int T, int h) {
  const int t = blockIdx.x;
  const long long row = ids[t];
  for (int i = threadIdx.x; i < h; i += blockDim.x)
    atomicAdd(dE + row * h + i, dx[(long long)t * h + i]);
}

// ---------------------------------------------------------- cross-entropy
// Per row of a bf16 logits chunk: lse, loss = lse - z[label] (label < 0 =>
// ignored), and in place dz = (softmax(z) - onehot) * grad_scale.
template <int THREADS>
__global__ void ce_fwd_bwd_kernel(__nv_bfloat16* __restrict__ z, long long ldz,
                                  const int32_t* __restrict__ labels, int V, float grad_scale,
                                  float* __restrict__ loss_sum, float* __restrict__ row_lse) {
  __shared__ float red[THREADS / 32];
  __shared__ float smax[THREADS / 32];
  const long long row = blockIdx.x;
  __nv_bfloat16* zr = z + row * ldz;
  const int label = labels[row];
  const bool vec = (V % 8 == 0) && (ldz % 8 == 0);
  // pass 1: running max + rescaled sum (online softmax per thread)
  float mx = -INFINITY, sum = 0.f;
  if (vec) {
    for (int c = threadIdx.x * 8; c < V; c += THREADS * 8) {
      float f[8];
      load8(zr + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (f[i] > mx) { sum *= __expf(mx - f[i]); mx = f[i]; }
        sum += __expf(f[i] - mx);
      }
    }
  } else {
    for (int c = threadIdx.x; c < V; c += THREADS) {
      const float f = bf2f(zr[c]);
      if (f > mx) { sum *= __expf(mx - f); mx = f; }
      sum += __expf(f - mx);
    }
  }
  // block max
  float m = mx;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x % 32 == 0) smax[threadIdx.x / 32] = m;
  __syncthreads();
  float gmax = -INFINITY;
#pragma unroll
  for (int i = 0; i < THREADS / 32; ++i) gmax = fmaxf(gmax, smax[i]);
  const float part = mx == -INFINITY ? 0.f : sum * __expf(mx - gmax);
  const float total = block_sum<THREADS>(part, red);
  const float lse = gmax + __logf(total);
  const float zl = label >= 0 ? bf2f(zr[label]) : 0.f;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (row_lse) row_lse[row] = lse;
    if (label >= 0 && loss_sum) atomicAdd(loss_sum, lse - zl);
  }
  // pass 2: dz in place
  const float s = label >= 0 ? grad_scale : 0.f;
  if (vec) {
    for (int c = threadIdx.x * 8; c < V; c += THREADS * 8) {
      float f[8];
      load8(zr + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = (__expf(f[i] - lse) - (c + i == label ? 1.f : 0.f)) * s;
      store8(zr + c, f);
    }
  } else {
    for (int c = threadIdx.x; c < V; c += THREADS) {
      const float f = bf2f(zr[c]);
      zr[c] = f2bf((__expf(f - lse) - (c == label ? 1.f : 0.f)) * s);
    }
  }
}

// ------------------------------------------------------------------- AdamW
// One streamed chunk of fp32 (master, m, v) in device memory, updated in
// place from the fp32 grad; writes the new bf16 weights. Decoupled weight
// decay (AdamW): p -= lr * (mhat / (sqrt(vhat) + eps) + wd * p).
__global__ void adamw_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ g, __nv_bfloat16* __restrict__ w16,
                             long long n, float lr, float b1, float b2, float eps, float wd,
                             float bc1, float bc2, float gscale) {
  const long long n4 = n / 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float* P = &pp.x;
    float* Mm = &mm.x;
    float* Vv = &vv.x;
    const float* G = &gg.x;
    __nv_bfloat16 o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float gk = G[k] * gscale;
      Mm[k] = b1 * Mm[k] + (1.f - b1) * gk;
      Vv[k] = b2 * Vv[k] + (1.f - b2) * gk * gk;
      const float upd = (Mm[k] / bc1) / (sqrtf(Vv[k] / bc2) + eps) + wd * P[k];
      P[k] -= lr * upd;
      o[k] = f2bf(P[k]);
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (w16) {
      uint2 u;
      __nv_bfloat162 lo2 = __halves2bfloat162(o[0], o[1]);
      __nv_bfloat162 hi2 = __halves2bfloat162(o[2], o[3]);
      u.x = *reinterpret_cast<uint32_t*>(&lo2);
      u.y = *reinterpret_cast<uint32_t*>(&hi2);
      reinterpret_cast<uint2*>(w16)[i] = u;
    }
  }
  // tail
  const long long tail0 = n4 * 4;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid < n - tail0) {
    const long long k = tail0 + tid;
    const float gk = g[k] * gscale;
    m[k] = b1 * m[k] + (1.f - b1) * gk;
    v[k] = b2 * v[k] + (1.f - b2) * gk * gk;
    p[k] -= lr * ((m[k] / bc1) / (sqrtf(v[k] / bc2) + eps) + wd * p[k]);
    if (w16) w16[k] = f2bf(p[k]);
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ a, __nv_bfloat16* __restrict__ b,
                                   long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    b[i] = f2bf(a[i]);
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ a, float* __restrict__ b,
                                   long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    b[i] = bf2f(a[i]);
}

__global__ void scale_bf16_kernel(__nv_bfloat16* __restrict__ a, long long n, float f) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = f2bf(bf2f(a[i]) * f);
}

__global__ void add_f32_kernel(float* __restrict__ a, const float* __restrict__ b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] += b[i];
}

int grid_for(long long work, int threads, int max_blocks = 148 * 8) {
  long long b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b < max_blocks ? b : max_blocks);
}

int status() { return cudaGetLastError() == cudaSuccess ? RP_OK : RP_E_CUDA; }

// one wave of resident QK_THREADS blocks (occupancy per device, cached), at
// most one block per token
template <auto Kern>
int wave_grid(int T) {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& g = cached[dev & 63];
  if (!g) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, Kern, QK_THREADS, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 1);
  }
  return T < g ? T : g;
}

}  // namespace
}  // namespace rp

using namespace rp;
#define RP_API extern "C" __attribute__((visibility("default")))

// 128 threads per row up to h = 4096, 256 above (h <= 8192); VPT vectors each
template <class Go, class F128_1, class F128_2, class F128_3, class F128_4, class F256_3,
          class F256_4>
void rn_dispatch(int h, Go go, F128_1 a, F128_2 b, F128_3 c, F128_4 d, F256_3 e, F256_4 f) {
  const int th = h <= 128 * 8 * 4 ? 128 : 256;
  const int vpt = (h + th * 8 - 1) / (th * 8);
  if (th == 128) {
    if (vpt <= 1) go(a, 128);
    else if (vpt <= 2) go(b, 128);
    else if (vpt <= 3) go(c, 128);
    else go(d, 128);
  } else {
    if (vpt <= 3) go(e, 256);
    else go(f, 256);
  }
}

RP_API int rp_rmsnorm_fwd(const void* x, int64_t ldx, const void* w, void* y, int64_t ldy,
                          float* rstd, int32_t rows, int32_t h, float eps, void* stream) {
  if (h % 8 || ldx % 8 || ldy % 8 || rows <= 0 || h > 256 * 8 * 4) return RP_E_INPUT;
  auto st = (cudaStream_t)stream;
  auto go = [&](auto kern, int th) {
    kern<<<rows, th, 0, st>>>((const __nv_bfloat16*)x, ldx, (const __nv_bfloat16*)w,
                              (__nv_bfloat16*)y, ldy, rstd, h, eps);
  };
  rn_dispatch(h, go, rmsnorm_fwd_kernel<128, 1>, rmsnorm_fwd_kernel<128, 2>,
              rmsnorm_fwd_kernel<128, 3>, rmsnorm_fwd_kernel<128, 4>,
              rmsnorm_fwd_kernel<256, 3>, rmsnorm_fwd_kernel<256, 4>);
  return status();
}

RP_API int rp_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd,
                          const float* dres, float* dx32, void* dx16, float* dw, int32_t rows,
                          int32_t h, void* stream) {
  if (h % 8 || rows <= 0 || h > 256 * 8 * 4) return RP_E_INPUT;
  auto st = (cudaStream_t)stream;
  // exactly the resident blocks (one wave); each walks rows grid-stride,
  // keeping dw in registers
  auto go = [&](auto kern, int th) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, th, 0) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    const int grid = rows < sms * per_sm ? rows : sms * per_sm;
    kern<<<grid, th, 0, st>>>((const __nv_bfloat16*)dy, (const __nv_bfloat16*)x,
                              (const __nv_bfloat16*)w, rstd, dres, dx32, (__nv_bfloat16*)dx16,
                              dw, rows, h);
  };
  // 256 threads above h = 1024: the row's dy / x / dres and the dw partials
  // live in registers, so fewer columns per thread keep occupancy up
  if (h <= 1024)
    go(rmsnorm_bwd_kernel<128, 1>, 128);
  else if (h <= 2048)
    go(rmsnorm_bwd_kernel<256, 1>, 256);
  else if (h <= 4096)
    go(rmsnorm_bwd_kernel<256, 2>, 256);
  else if (h <= 6144)
    go(rmsnorm_bwd_kernel<256, 3>, 256);
  else
    go(rmsnorm_bwd_kernel<256, 4>, 256);
  return status();
}

RP_API int rp_qk_norm_rope_fwd(const void* qkv, int64_t ld, int32_t nq, int32_t nk,
                               int32_t head_dim, const void* qw, const void* kw,
                               const float* cos_sin, int32_t seq, void* q_out, void* k_out,
                               float* rstd_q, float* rstd_k, int32_t T, float eps,
                               void* stream) {
  if (ld % 8 || T % 128 || T <= 0) return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  if (head_dim == 128)
    qk_norm_rope_fwd_kernel<128><<<wave_grid<qk_norm_rope_fwd_kernel<128>>(T), QK_THREADS, 0, s>>>(
        (const __nv_bfloat16*)qkv, ld, nq, nk, (const __nv_bfloat16*)qw, (const __nv_bfloat16*)kw,
        (const float2*)cos_sin, seq, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_out, rstd_q, rstd_k,
        T, eps);
  else if (head_dim == 64)
    qk_norm_rope_fwd_kernel<64><<<wave_grid<qk_norm_rope_fwd_kernel<64>>(T), QK_THREADS, 0, s>>>(
        (const __nv_bfloat16*)qkv, ld, nq, nk, (const __nv_bfloat16*)qw, (const __nv_bfloat16*)kw,
        (const float2*)cos_sin, seq, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_out, rstd_q, rstd_k,
        T, eps);
  else
    return RP_E_INPUT;
  return status();
}

RP_API int rp_qk_norm_rope_bwd(const void* dq, const void* dk, const void* qkv, int64_t ld,
                               int32_t nq, int32_t nk, int32_t head_dim, const void* qw,
                               const void* kw, const float* rstd_q, const float* rstd_k,
                               const float* cos_sin, int32_t seq, void* dqkv, int64_t ldd,
                               float* dqw, float* dkw, int32_t T, void* stream) {
  if (ld % 8 || ldd % 8 || T % 128 || T <= 0) return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  if (head_dim == 128)
    qk_norm_rope_bwd_kernel<128><<<wave_grid<qk_norm_rope_bwd_kernel<128>>(T), QK_THREADS, 0, s>>>(
        (const __nv_bfloat16*)dq, (const __nv_bfloat16*)dk, (const __nv_bfloat16*)qkv, ld, nq, nk,
        (const __nv_bfloat16*)qw, (const __nv_bfloat16*)kw, rstd_q, rstd_k, (const float2*)cos_sin,
        seq, (__nv_bfloat16*)dqkv, ldd, dqw, dkw, T);
  else if (head_dim == 64)
    qk_norm_rope_bwd_kernel<64><<<wave_grid<qk_norm_rope_bwd_kernel<64>>(T), QK_THREADS, 0, s>>>(
        (const __nv_bfloat16*)dq, (const __nv_bfloat16*)dk, (const __nv_bfloat16*)qkv, ld, nq, nk,
        (const __nv_bfloat16*)qw, (const __nv_bfloat16*)kw, rstd_q, rstd_k, (const float2*)cos_sin,
        seq, (__nv_bfloat16*)dqkv, ldd, dqw, dkw, T);
  else
    return RP_E_INPUT;
  return status();
}

RP_API int rp_swiglu_fwd(const void* gu, void* act, int64_t T, int32_t m, void* stream) {
  if (m % 8) return RP_E_INPUT;
  if (T <= 0) return RP_OK;
  swiglu_fwd_kernel<<<(unsigned)T, 256, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)gu, (__nv_bfloat16*)act, m);
  return status();
}

RP_API int rp_swiglu_bwd(const void* dact, const void* gu, void* dgu, int64_t T, int32_t m,
                         void* stream) {
  if (m % 8) return RP_E_INPUT;
  if (T <= 0) return RP_OK;
  swiglu_bwd_kernel<<<(unsigned)T, 256, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)dact, (const __nv_bfloat16*)gu, (__nv_bfloat16*)dgu, m);
  return status();
}

RP_API int rp_embed_fwd(const int32_t* ids, const void* table, void* out, int32_t T, int32_t h,
                        void* stream) {
  if (h % 8) return RP_E_INPUT;
  embed_fwd_kernel<<<T, 128, 0, (cudaStream_t)stream>>>(ids, (const __nv_bfloat16*)table,
                                                        (__nv_bfloat16*)out, T, h);
  return status();
}

RP_API int rp_embed_bwd(const int32_t* ids, const float* dx, float* dE, int32_t T, int32_t h,
                        void* stream) {
  embed_bwd_kernel<<<T, 256, 0, (cudaStream_t)stream>>>(ids, dx, dE, T, h);
  return status();
}

RP_API int rp_ce_fwd_bwd(void* logits, int64_t ld, const int32_t* labels, int32_t rows,
                         int32_t V, float grad_scale, float* loss_sum, float* row_lse,
                         void* stream) {
  if (rows <= 0) return RP_OK;
  ce_fwd_bwd_kernel<512><<<rows, 512, 0, (cudaStream_t)stream>>>(
      (__nv_bfloat16*)logits, ld, labels, V, grad_scale, loss_sum, row_lse);
  return status();
}

RP_API int rp_adamw(float* master, float* m, float* v, const float* grad, void* w16, int64_t n,
                    const rp_adam_hparams_t* hp, int32_t step, void* stream) {
  if (!hp || step < 1 || (reinterpret_cast<uintptr_t>(master) & 15) ||
      (reinterpret_cast<uintptr_t>(m) & 15) || (reinterpret_cast<uintptr_t>(v) & 15) ||
      (reinterpret_cast<uintptr_t>(grad) & 15) || (w16 && (reinterpret_cast<uintptr_t>(w16) & 7)))
    return RP_E_INPUT;
  const float bc1 = 1.f - powf(hp->beta1, (float)step);
  const float bc2 = 1.f - powf(hp->beta2, (float)step);
  adamw_kernel<<<grid_for(n / 4 + 4, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      master, m, v, grad, (__nv_bfloat16*)w16, n, hp->lr, hp->beta1, hp->beta2, hp->eps,
      hp->weight_decay, bc1, bc2, hp->grad_scale);
  return status();
}

RP_API int rp_f32_to_bf16(const float* a, void* b, int64_t n, void* stream) {
  f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(a, (__nv_bfloat16*)b, n);
  return status();
}

RP_API int rp_bf16_to_f32(const void* a, float* b, int64_t n, void* stream) {
  bf16_to_f32_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)a,
                                                                          b, n);
  return status();
}

RP_API int rp_scale_bf16(void* a, int64_t n, float f, void* stream) {
  if (n <= 0) return RP_OK;
  scale_bf16_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>((__nv_bfloat16*)a, n, f);
  return status();
}

RP_API int rp_add_f32(float* a, const float* b, int64_t n, void* stream) {
  add_f32_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(a, b, n);
  return status();
}

// ---------------------------------------------------------------- init
namespace rp {
namespace {
__device__ __forceinline__ uint32_t mix32(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return static_cast<uint32_t>(x);
}
// Deterministic N(0, std) (Box-Muller on a counter hash), rounded to bf16;
// writes the bf16 value and (optionally) its exact fp32 widening.
__global__ void init_normal_kernel(float* __restrict__ f32, uint16_t* __restrict__ b16,
                                   long long n, unsigned long long seed, float std) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint32_t a = mix32(seed * 0x9E3779B97F4A7C15ULL + 2 * (unsigned long long)i);
    const uint32_t b = mix32(seed * 0x9E3779B97F4A7C15ULL + 2 * (unsigned long long)i + 1);
    const float u1 = (a + 1.0f) * 2.3283064e-10f, u2 = b * 2.3283064e-10f;
    const float z = sqrtf(-2.f * __logf(u1)) * __cosf(6.2831853f * u2) * std;
    const __nv_bfloat16 hb = __float2bfloat16_rn(z);
    if (f32) f32[i] = __bfloat162float(hb);
    b16[i] = *reinterpret_cast<const uint16_t*>(&hb);
  }
}
__global__ void fill_kernel(float* __restrict__ f32, uint16_t* __restrict__ b16, long long n,
                            float value) {
  const __nv_bfloat16 hb = __float2bfloat16_rn(value);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (f32) f32[i] = value;
    b16[i] = *reinterpret_cast<const uint16_t*>(&hb);
  }
}
}  // namespace
}  // namespace rp

RP_API int rp_init_normal(float* f32, void* b16, int64_t n, uint64_t seed, float std,
                          void* stream) {
  init_normal_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      f32, (uint16_t*)b16, n, seed, std);
  return status();
}

RP_API int rp_fill(float* f32, void* b16, int64_t n, float value, void* stream) {
  fill_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(f32, (uint16_t*)b16, n,
                                                                           value);
  return status();
}
