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

#include <cstdio>

#include "kernels/launch_util.h"
#include "kernels/sm100.cuh"
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

// bf16x2 word <-> float2 (low half = .x)
__device__ __forceinline__ float2 bf2x2(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}
__device__ __forceinline__ uint32_t pack_bf16x2_rn(float2 v) {
  const __nv_bfloat162 b = __floats2bfloat162_rn(v.x, v.y);
  return *reinterpret_cast<const uint32_t*>(&b);
}
__device__ __forceinline__ void unpack4(const uint2& u, float (&f)[4]) {
  const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) f[i] = bf2f(b[i]);
}
__device__ __forceinline__ void store4(__nv_bfloat16* p, const float (&f)[4]) {
  uint2 u;
  __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = f2bf(f[i]);
  *reinterpret_cast<uint2*>(p) = u;
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

// The same backward with the row's operands staged by the copy engine: one
// wave of persistent blocks, each with a ring of RN_ST rows in shared memory
// ([dy bf16 | x bf16 | dres fp32 | the 16-byte rstd group of the row]) filled
// by 1-D bulk copies on an mbarrier per slot, so the bytes in flight are not
// bounded by the registers that hold them (the register version keeps one
// row per block in flight, profiles/r02n_step_breakdown_8b.txt: 3.7 TB/s in
// step). The per-thread column assignment, the dot-product order and the
// output arithmetic are the register version's (the compiler's fp32
// contraction can still differ in the last bit).
constexpr int RN_ST = 2;
#ifndef RN_STAGED  // -DRN_STAGED=0: register version only (same-box A/B builds)
#define RN_STAGED 1
#endif
template <int RN_THREADS, int VPT>
__global__ void __launch_bounds__(RN_THREADS)
    rmsnorm_bwd_staged_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                              const __nv_bfloat16* __restrict__ w, const float* __restrict__ rstd,
                              const float* __restrict__ dres, float* __restrict__ dx32,
                              __nv_bfloat16* __restrict__ dx16, float* __restrict__ dw, int rows,
                              int h) {
  using namespace sm100;
  extern __shared__ __align__(128) uint8_t rsm[];
  __shared__ float red[2][RN_THREADS / 32];
  const int slot_bytes = h * (dres ? 8 : 4) + 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(rsm + RN_ST * slot_bytes);
  auto issue = [&](int row, int s) {
    uint8_t* slot = rsm + s * slot_bytes;
    const long long off = (long long)row * h;
    mbar_arrive_expect_tx(&full[s], slot_bytes);
    bulk_load_1d(slot, dy + off, h * 2, &full[s]);
    bulk_load_1d(slot + h * 2, x + off, h * 2, &full[s]);
    if (dres) bulk_load_1d(slot + h * 4, dres + off, h * 4, &full[s]);
    bulk_load_1d(slot + slot_bytes - 16, rstd + (row & ~3), 16, &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < RN_ST; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    for (int s = 0; s < RN_ST; ++s)
      if (blockIdx.x + s * gridDim.x < rows) issue(blockIdx.x + s * gridDim.x, s);
  }
  uint4 wv[VPT];
  float dwa[VPT][8];
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int c = (threadIdx.x + j * RN_THREADS) * 8;
    wv[j] = c < h ? *reinterpret_cast<const uint4*>(w + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) dwa[j][i] = 0.f;
  }
  __syncthreads();
  int par = 0, it = 0;
  for (int row = blockIdx.x; row < rows; row += gridDim.x, par ^= 1, ++it) {
    const int s = it % RN_ST;
    mbar_wait(&full[s], (it / RN_ST) & 1);
    const uint8_t* slot = rsm + s * slot_bytes;
    const __nv_bfloat16* dys = reinterpret_cast<const __nv_bfloat16*>(slot);
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(slot + h * 2);
    const float* ds = reinterpret_cast<const float*>(slot + h * 4);
    const long long off = (long long)row * h;
    const float r = reinterpret_cast<const float*>(slot + slot_bytes - 16)[row & 3];
    // dy / x are read from the slot twice (before and after the row
    // reduction) instead of being held in registers across it
    float dot = 0.f;
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int c = (threadIdx.x + j * RN_THREADS) * 8;
      float a[8], b[8], g[8];
      unpack8(c < h ? *reinterpret_cast<const uint4*>(dys + c) : make_uint4(0, 0, 0, 0), a);
      unpack8(c < h ? *reinterpret_cast<const uint4*>(xs + c) : make_uint4(0, 0, 0, 0), b);
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
      unpack8(*reinterpret_cast<const uint4*>(dys + c), a);
      unpack8(*reinterpret_cast<const uint4*>(xs + c), b);
      unpack8(wv[j], g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = b[i] * r;
        o[i] = r * (a[i] * g[i] - xh * mean);
        dwa[j][i] += a[i] * xh;
      }
      if (dres) {
        const float4 d0 = *reinterpret_cast<const float4*>(ds + c);
        const float4 d1 = *reinterpret_cast<const float4*>(ds + c + 4);
        o[0] += d0.x; o[1] += d0.y; o[2] += d0.z; o[3] += d0.w;
        o[4] += d1.x; o[5] += d1.y; o[6] += d1.z; o[7] += d1.w;
      }
      if (dx32) {
        *reinterpret_cast<float4*>(dx32 + off + c) = make_float4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<float4*>(dx32 + off + c + 4) = make_float4(o[4], o[5], o[6], o[7]);
      }
      if (dx16) store8(dx16 + off + c, o);
    }
    __syncthreads();  // slot s consumed
    if (threadIdx.x == 0 && row + RN_ST * gridDim.x < rows) issue(row + RN_ST * gridDim.x, s);
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
// A head of HD elements is handled by TPH = HD/8 consecutive lanes; lane
// `sub` owns the rotate_half PAIRS (e, e + HD/2) for e in [4 sub, 4 sub + 4),
// so the rotation needs no shuffles (only the per-head RMS reduces over the
// TPH lanes) and a lane's (cos, sin) are 4 float2 kept in registers for the
// token.
//
// Bytes in flight come from the copy engine, not from registers: one wave of
// persistent blocks walks tokens, and one thread per block keeps a ring of
// QK_STAGES tokens in shared memory filled with 1-D bulk copies
// (cp.async.bulk, an mbarrier per slot): a token's q|k head slice of the qkv
// row (contiguous), its (cos, sin) row and, backward, the dq / dk rows and
// the per-head rstd. The block's threads (qk_block_threads: QK_NB passes
// cover a token's heads) compute from the slot, store straight to global,
// and a __syncthreads hands the slot back to the producer for the token
// QK_STAGES steps ahead. The round-1/2 kernels held QK_NB 16-byte loads per
// thread in registers (8 contiguous elements, partner via lane ^ TPH/2):
// register-limited occupancy, 12 shuffles per 8 elements, one memory round
// trip per token (profiles/r02g_ncu_full.json, profiles/r02_qk_ab.jsonl).
#ifndef QK_NB
#define QK_NB 4
#endif
constexpr int QK_MAX_THREADS = 512;
#ifndef QK_STAGES_FWD
#define QK_STAGES_FWD 2
#endif
#ifndef QK_STAGES_BWD
#define QK_STAGES_BWD 2
#endif

template <int HD>
__host__ __device__ constexpr int qk_tph() { return HD / 8; }

template <int HD>
int qk_block_threads(int heads, int nb) {
  const int slots = heads * qk_tph<HD>();
  int bt = (slots + nb - 1) / nb;
  bt = (bt + 31) / 32 * 32;
  return bt < QK_MAX_THREADS ? bt : QK_MAX_THREADS;
}

__host__ __device__ constexpr int qk_align16(int b) { return (b + 15) / 16 * 16; }

// shared-memory slot of one token: [x: heads*HD bf16 | cs: HD/2 float2] (fwd),
// [g: heads*HD bf16 (dq row, dk row) | x | cs | rstd: heads fp32] (bwd)
struct QkSlot {
  int x, cs, g, rstd, bytes;
};
template <int HD>
__host__ __device__ QkSlot qk_slot(int heads, bool bwd) {
  QkSlot q;
  const int row = heads * HD * 2;
  q.g = 0;
  q.x = bwd ? row : 0;
  q.cs = q.x + row;
  q.rstd = q.cs + qk_align16(HD / 2 * 8);
  q.bytes = (q.rstd + (bwd ? qk_align16(heads * 4) : 0) + 127) / 128 * 128;
  return q;
}

template <int HD>
__global__ void __launch_bounds__(QK_MAX_THREADS)
    qk_norm_rope_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, long long ld, int nq, int nk,
                            const __nv_bfloat16* __restrict__ qw,
                            const __nv_bfloat16* __restrict__ kw, const float2* __restrict__ cs,
                            int seq, __nv_bfloat16* __restrict__ qo, __nv_bfloat16* __restrict__ ko,
                            float* __restrict__ rstd_q, float* __restrict__ rstd_k, int T,
                            float eps) {
  using namespace sm100;
  constexpr int TPH = qk_tph<HD>(), HALF = HD / 2, ST = QK_STAGES_FWD;
  extern __shared__ __align__(128) uint8_t qsm[];
  const int heads = nq + nk;
  const QkSlot L = qk_slot<HD>(heads, false);
  uint64_t* full = reinterpret_cast<uint64_t*>(qsm + ST * L.bytes);
  const int sub = threadIdx.x % TPH, h0 = threadIdx.x / TPH, hstep = blockDim.x / TPH;
  const bool lo = sub < TPH / 2;
  auto issue = [&](int t, int s) {
    uint8_t* slot = qsm + s * L.bytes;
    mbar_arrive_expect_tx(&full[s], heads * HD * 2 + HALF * 8);
    bulk_load_1d(slot + L.x, qkv + (long long)t * ld, heads * HD * 2, &full[s]);
    bulk_load_1d(slot + L.cs, cs + (long long)(t % seq) * HALF, HALF * 8, &full[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    for (int s = 0; s < ST; ++s)
      if (blockIdx.x + s * gridDim.x < T) issue(blockIdx.x + s * gridDim.x, s);
  }
  __syncthreads();
  const int e0 = sub * 4;  // this lane's pairs (e0 + k, e0 + k + HALF), k < 4
  float2 wq2l[2], wq2h[2], wk2l[2], wk2h[2];  // norm weights, converted once
  {
    const uint2 a = *reinterpret_cast<const uint2*>(qw + e0), b = *reinterpret_cast<const uint2*>(qw + HALF + e0);
    const uint2 c = *reinterpret_cast<const uint2*>(kw + e0), d = *reinterpret_cast<const uint2*>(kw + HALF + e0);
    wq2l[0] = bf2x2(a.x), wq2l[1] = bf2x2(a.y), wq2h[0] = bf2x2(b.x), wq2h[1] = bf2x2(b.y);
    wk2l[0] = bf2x2(c.x), wk2l[1] = bf2x2(c.y), wk2h[0] = bf2x2(d.x), wk2h[1] = bf2x2(d.y);
  }
  int i = 0;
  for (int t = blockIdx.x; t < T; t += gridDim.x, ++i) {
    const int s = i % ST;
    mbar_wait(&full[s], (i / ST) & 1);
    const uint8_t* slot = qsm + s * L.bytes;
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(slot + L.x);
    const float4* c4 = reinterpret_cast<const float4*>(slot + L.cs) + e0 / 2;
    const float4 ca = c4[0], cb = c4[1];  // (cos, sin) of pairs e0 .. e0+3
    const float2 cos2[2] = {make_float2(ca.x, ca.z), make_float2(cb.x, cb.z)};
    const float2 sin2[2] = {make_float2(ca.y, ca.w), make_float2(cb.y, cb.w)};
    const float2 nsin2[2] = {make_float2(-ca.y, -ca.w), make_float2(-cb.y, -cb.w)};
    __nv_bfloat16* qrow = qo + (long long)t * nq * HD;
    __nv_bfloat16* krow = ko + (long long)t * nk * HD;
    float* rq_row = rstd_q + (long long)t * nq;
    float* rk_row = rstd_k + (long long)t * nk;
    // every lane runs every pass (the RMS shuffles are warp-wide); lanes
    // whose head is past the end store nothing
    for (int hb = 0; hb < heads; hb += hstep) {  // block-uniform
      const int hh = hb + h0;
      const bool act = hh < heads;
      const bool is_q = hh < nq;
      // lanes past the last head recompute the last head (no zero paths;
      // their 16-lane reductions never mix with a stored head's)
      const int hr = act ? hh : heads - 1;
      // packed fp32x2 math (FFMA2 / FMUL2): element pairs (e0+2j, e0+2j+1)
      const uint2 xl = *reinterpret_cast<const uint2*>(xs + hr * HD + e0);
      const uint2 xh = *reinterpret_cast<const uint2*>(xs + hr * HD + HALF + e0);
      const float2 lo[2] = {bf2x2(xl.x), bf2x2(xl.y)}, hi[2] = {bf2x2(xh.x), bf2x2(xh.y)};
      float2 acc = __fmul2_rn(lo[0], lo[0]);
      acc = __ffma2_rn(lo[1], lo[1], acc);
      acc = __ffma2_rn(hi[0], hi[0], acc);
      acc = __ffma2_rn(hi[1], hi[1], acc);
      float ss = acc.x + acc.y;
#pragma unroll
      for (int o = TPH / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float r = rsqrtf(ss / HD + eps);
      const float2 r2 = make_float2(r, r);
      float ol[4], oh[4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float2 wl = is_q ? wq2l[j] : wk2l[j], wh = is_q ? wq2h[j] : wk2h[j];
        // the normalised value rounded to bf16 (HF computes the norm in bf16)
        const float2 nl = bf2x2(pack_bf16x2_rn(__fmul2_rn(wl, __fmul2_rn(lo[j], r2))));
        const float2 nh = bf2x2(pack_bf16x2_rn(__fmul2_rn(wh, __fmul2_rn(hi[j], r2))));
        const float2 l2 = __ffma2_rn(nl, cos2[j], __fmul2_rn(nh, nsin2[j]));  // x1 cos - x2 sin
        const float2 h2 = __ffma2_rn(nh, cos2[j], __fmul2_rn(nl, sin2[j]));   // x2 cos + x1 sin
        ol[2 * j] = l2.x, ol[2 * j + 1] = l2.y;
        oh[2 * j] = h2.x, oh[2 * j + 1] = h2.y;
      }
      if (!act) continue;
      __nv_bfloat16* dst = is_q ? qrow + hh * HD : krow + (hh - nq) * HD;
      store4(dst + e0, ol);
      store4(dst + HALF + e0, oh);
      if (sub == 0) (is_q ? rq_row[hh] : rk_row[hh - nq]) = r;
    }
    __syncthreads();  // slot s consumed
    if (threadIdx.x == 0 && t + ST * gridDim.x < T) issue(t + ST * gridDim.x, s);
  }
}

// Backward: undo the rotation (R^T), then per-head RMSNorm backward;
// dqkv[:, q/k slots] = dx; dqw/dkw[HD] += sum(dn * xhat) (registers -> smem
// -> one atomic per column per block). rstd_bulk: nq, nk multiples of 4 (the
// rstd rows are bulk-copied); otherwise rstd is read from global.
template <int HD>
__global__ void __launch_bounds__(QK_MAX_THREADS)
    qk_norm_rope_bwd_kernel(const __nv_bfloat16* __restrict__ dq, const __nv_bfloat16* __restrict__ dk,
                            const __nv_bfloat16* __restrict__ qkv, long long ld, int nq, int nk,
                            const __nv_bfloat16* __restrict__ qw,
                            const __nv_bfloat16* __restrict__ kw, const float* __restrict__ rstd_q,
                            const float* __restrict__ rstd_k, const float2* __restrict__ cs, int seq,
                            __nv_bfloat16* __restrict__ dqkv, long long ldd, float* __restrict__ dqw,
                            float* __restrict__ dkw, int T, int rstd_bulk) {
  using namespace sm100;
  constexpr int TPH = qk_tph<HD>(), HALF = HD / 2, ST = QK_STAGES_BWD;
  extern __shared__ __align__(128) uint8_t qsm[];
  __shared__ float sq[HD], sk[HD];
  const int heads = nq + nk;
  const QkSlot L = qk_slot<HD>(heads, true);
  uint64_t* full = reinterpret_cast<uint64_t*>(qsm + ST * L.bytes);
  const int sub = threadIdx.x % TPH, h0 = threadIdx.x / TPH, hstep = blockDim.x / TPH;
  const bool lo = sub < TPH / 2;
  auto issue = [&](int t, int s) {
    uint8_t* slot = qsm + s * L.bytes;
    mbar_arrive_expect_tx(&full[s], 2 * heads * HD * 2 + HALF * 8 + (rstd_bulk ? heads * 4 : 0));
    bulk_load_1d(slot + L.g, dq + (long long)t * nq * HD, nq * HD * 2, &full[s]);
    bulk_load_1d(slot + L.g + nq * HD * 2, dk + (long long)t * nk * HD, nk * HD * 2, &full[s]);
    bulk_load_1d(slot + L.x, qkv + (long long)t * ld, heads * HD * 2, &full[s]);
    bulk_load_1d(slot + L.cs, cs + (long long)(t % seq) * HALF, HALF * 8, &full[s]);
    if (rstd_bulk) {
      bulk_load_1d(slot + L.rstd, rstd_q + (long long)t * nq, nq * 4, &full[s]);
      bulk_load_1d(slot + L.rstd + nq * 4, rstd_k + (long long)t * nk, nk * 4, &full[s]);
    }
  };
  for (int k = threadIdx.x; k < HD; k += blockDim.x) sq[k] = sk[k] = 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    for (int s = 0; s < ST; ++s)
      if (blockIdx.x + s * gridDim.x < T) issue(blockIdx.x + s * gridDim.x, s);
  }
  __syncthreads();
  const int e0 = sub * 4;  // this lane's pairs (e0 + k, e0 + k + HALF), k < 4
  float2 wq2l[2], wq2h[2], wk2l[2], wk2h[2];  // norm weights, converted once
  {
    const uint2 a = *reinterpret_cast<const uint2*>(qw + e0), b = *reinterpret_cast<const uint2*>(qw + HALF + e0);
    const uint2 c = *reinterpret_cast<const uint2*>(kw + e0), d = *reinterpret_cast<const uint2*>(kw + HALF + e0);
    wq2l[0] = bf2x2(a.x), wq2l[1] = bf2x2(a.y), wq2h[0] = bf2x2(b.x), wq2h[1] = bf2x2(b.y);
    wk2l[0] = bf2x2(c.x), wk2l[1] = bf2x2(c.y), wk2h[0] = bf2x2(d.x), wk2h[1] = bf2x2(d.y);
  }
  // dw partials, element pairs: [0, 2) = lo pairs (e0 + 2j, +1), [2, 4) = hi pairs
  float2 aq[4], ak[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) aq[k] = ak[k] = make_float2(0.f, 0.f);
  int i = 0;
  for (int t = blockIdx.x; t < T; t += gridDim.x, ++i) {
    const int s = i % ST;
    mbar_wait(&full[s], (i / ST) & 1);
    const uint8_t* slot = qsm + s * L.bytes;
    const __nv_bfloat16* gs = reinterpret_cast<const __nv_bfloat16*>(slot + L.g);
    const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(slot + L.x);
    const float* rs = reinterpret_cast<const float*>(slot + L.rstd);
    const float4* c4 = reinterpret_cast<const float4*>(slot + L.cs) + e0 / 2;
    const float4 ca = c4[0], cb = c4[1];
    const float2 cos2[2] = {make_float2(ca.x, ca.z), make_float2(cb.x, cb.z)};
    const float2 sin2[2] = {make_float2(ca.y, ca.w), make_float2(cb.y, cb.w)};
    const float2 nsin2[2] = {make_float2(-ca.y, -ca.w), make_float2(-cb.y, -cb.w)};
    __nv_bfloat16* drow = dqkv + (long long)t * ldd;
    for (int hb = 0; hb < heads; hb += hstep) {  // block-uniform (shuffles)
      const int hh = hb + h0;
      const bool act = hh < heads;
      const bool is_q = hh < nq;
      // lanes past the last head recompute the last head and store nothing
      // (their dw contributions are masked below)
      const int hr = act ? hh : heads - 1;
      const bool rq = hr < nq;
      const float r = rstd_bulk ? rs[hr] : rq ? rstd_q[(long long)t * nq + hr] : rstd_k[(long long)t * nk + (hr - nq)];
      // packed fp32x2 math (FFMA2 / FMUL2) over element pairs (e0+2j, e0+2j+1)
      const uint2 ugl = *reinterpret_cast<const uint2*>(gs + hr * HD + e0);
      const uint2 ugh = *reinterpret_cast<const uint2*>(gs + hr * HD + HALF + e0);
      const uint2 uxl = *reinterpret_cast<const uint2*>(xs + hr * HD + e0);
      const uint2 uxh = *reinterpret_cast<const uint2*>(xs + hr * HD + HALF + e0);
      const float2 gl[2] = {bf2x2(ugl.x), bf2x2(ugl.y)}, gh[2] = {bf2x2(ugh.x), bf2x2(ugh.y)};
      const float2 r2 = make_float2(r, r);
      float2 xl[2] = {__fmul2_rn(bf2x2(uxl.x), r2), __fmul2_rn(bf2x2(uxl.y), r2)};  // xhat
      float2 xh[2] = {__fmul2_rn(bf2x2(uxh.x), r2), __fmul2_rn(bf2x2(uxh.y), r2)};
      float2 gxl[2], gxh[2], dnl[2], dnh[2];
      float2 dacc = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        dnl[j] = __ffma2_rn(gl[j], cos2[j], __fmul2_rn(gh[j], sin2[j]));   // R^T
        dnh[j] = __ffma2_rn(gh[j], cos2[j], __fmul2_rn(gl[j], nsin2[j]));
        gxl[j] = __fmul2_rn(dnl[j], is_q ? wq2l[j] : wk2l[j]);
        gxh[j] = __fmul2_rn(dnh[j], is_q ? wq2h[j] : wk2h[j]);
        dacc = __ffma2_rn(gxl[j], xl[j], dacc);
        dacc = __ffma2_rn(gxh[j], xh[j], dacc);
      }
      if (act) {
        float2* acc = is_q ? aq : ak;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          acc[j] = __ffma2_rn(dnl[j], xl[j], acc[j]);
          acc[2 + j] = __ffma2_rn(dnh[j], xh[j], acc[2 + j]);
        }
      }
      float dot = dacc.x + dacc.y;
#pragma unroll
      for (int o = TPH / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      const float2 nmean = make_float2(-dot / HD, -dot / HD);
      if (act) {
        uint2 ol, oh;
        ol.x = pack_bf16x2_rn(__fmul2_rn(r2, __ffma2_rn(xl[0], nmean, gxl[0])));
        ol.y = pack_bf16x2_rn(__fmul2_rn(r2, __ffma2_rn(xl[1], nmean, gxl[1])));
        oh.x = pack_bf16x2_rn(__fmul2_rn(r2, __ffma2_rn(xh[0], nmean, gxh[0])));
        oh.y = pack_bf16x2_rn(__fmul2_rn(r2, __ffma2_rn(xh[1], nmean, gxh[1])));
        __nv_bfloat16* dst = drow + hh * HD;
        *reinterpret_cast<uint2*>(dst + e0) = ol;
        *reinterpret_cast<uint2*>(dst + HALF + e0) = oh;
      }
    }
    __syncthreads();  // slot s consumed
    if (threadIdx.x == 0 && t + ST * gridDim.x < T) issue(t + ST * gridDim.x, s);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    atomicAdd(&sq[e0 + 2 * j], aq[j].x);
    atomicAdd(&sq[e0 + 2 * j + 1], aq[j].y);
    atomicAdd(&sq[HALF + e0 + 2 * j], aq[2 + j].x);
    atomicAdd(&sq[HALF + e0 + 2 * j + 1], aq[2 + j].y);
    atomicAdd(&sk[e0 + 2 * j], ak[j].x);
    atomicAdd(&sk[e0 + 2 * j + 1], ak[j].y);
    atomicAdd(&sk[HALF + e0 + 2 * j], ak[2 + j].x);
    atomicAdd(&sk[HALF + e0 + 2 * j + 1], ak[2 + j].y);
  }
  __syncthreads();
  if (dqw && dkw)  // null: frozen norm weights (LoRA)
    for (int k = threadIdx.x; k < HD; k += blockDim.x) {
      atomicAdd(dqw + k, sq[k]);
      atomicAdd(dkw + k, sk[k]);
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

// a failed launch names its CUDA error on stderr (the caller only sees RP_E_CUDA)
int status() {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return RP_OK;
  std::fprintf(stderr, "rp elementwise kernel launch: %s\n", cudaGetErrorString(e));
  return RP_E_CUDA;
}

// one wave of resident bt-thread blocks of kern with `smem` dynamic shared
// memory (occupancy per (device, kernel, bt, smem), the last configuration
// asked per device and kernel type cached), at most one block per token
template <class K>
int qk_wave_grid(K* kern, int bt, int smem, int T) {
  struct Entry {
    const void* kern = nullptr;
    int bt = 0, smem = -1, grid = 0;
  };
  static thread_local Entry cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  Entry& e = cached[dev & 63];
  if (e.kern != reinterpret_cast<const void*>(kern) || e.bt != bt || e.smem != smem) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, bt, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e.grid = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 1);
    e.kern = reinterpret_cast<const void*>(kern), e.bt = bt, e.smem = smem;
  }
  return T < e.grid ? T : e.grid;
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
  auto go = [&](auto kern, int th, int smem) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, th, smem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    const int grid = rows < sms * per_sm ? rows : sms * per_sm;
    kern<<<grid, th, smem, st>>>((const __nv_bfloat16*)dy, (const __nv_bfloat16*)x,
                                 (const __nv_bfloat16*)w, rstd, dres, dx32, (__nv_bfloat16*)dx16,
                                 dw, rows, h);
  };
  // staged (bulk-copy ring) when the operands allow 16-byte bulk copies:
  // 16-byte aligned bases, rstd readable in 16-byte groups (rows % 4 == 0)
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool staged = RN_STAGED && h >= 1024 && rows % 4 == 0 && al(dy) && al(x) && al(rstd) && (!dres || al(dres));
  if (staged) {
    const int smem = RN_ST * (h * (dres ? 8 : 4) + 16) + RN_ST * 8;
    auto sgo = [&](auto kern, int th) {
      if (!ensure_smem_t(kern, smem)) return false;
      go(kern, th, smem);
      return true;
    };
    bool ok;
    if (h <= 2048)
      ok = sgo(rmsnorm_bwd_staged_kernel<256, 1>, 256);
    else if (h <= 4096)
      ok = sgo(rmsnorm_bwd_staged_kernel<256, 2>, 256);
    else if (h <= 6144)
      ok = sgo(rmsnorm_bwd_staged_kernel<256, 3>, 256);
    else
      ok = sgo(rmsnorm_bwd_staged_kernel<256, 4>, 256);
    if (!ok) return RP_E_INPUT;
    return status();
  }
  // 256 threads above h = 1024: the row's dy / x / dres and the dw partials
  // live in registers, so fewer columns per thread keep occupancy up
  if (h <= 1024)
    go(rmsnorm_bwd_kernel<128, 1>, 128, 0);
  else if (h <= 2048)
    go(rmsnorm_bwd_kernel<256, 1>, 256, 0);
  else if (h <= 4096)
    go(rmsnorm_bwd_kernel<256, 2>, 256, 0);
  else if (h <= 6144)
    go(rmsnorm_bwd_kernel<256, 3>, 256, 0);
  else
    go(rmsnorm_bwd_kernel<256, 4>, 256, 0);
  return status();
}

// bulk copies need 16-byte aligned sources: ld % 8 (bf16), 16-byte aligned
// base pointers (row strides nq*HD, nk*HD are multiples of 8 elements)
static bool qk_aligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

RP_API int rp_qk_norm_rope_fwd(const void* qkv, int64_t ld, int32_t nq, int32_t nk,
                               int32_t head_dim, const void* qw, const void* kw,
                               const float* cos_sin, int32_t seq, void* q_out, void* k_out,
                               float* rstd_q, float* rstd_k, int32_t T, float eps,
                               void* stream) {
  if (ld % 8 || T % 128 || T <= 0 || nq <= 0 || nk <= 0 || seq <= 0) return RP_E_INPUT;
  if (!qk_aligned(qkv) || !qk_aligned(cos_sin) || !qk_aligned(qw) || !qk_aligned(kw) ||
      !qk_aligned(q_out) || !qk_aligned(k_out))
    return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  auto go = [&](auto kern, int bt, QkSlot L) -> int {
    const int smem = QK_STAGES_FWD * L.bytes + QK_STAGES_FWD * 8;
    if (!ensure_smem_t(kern, smem)) return RP_E_INPUT;
    kern<<<qk_wave_grid(kern, bt, smem, T), bt, smem, s>>>(
        (const __nv_bfloat16*)qkv, ld, nq, nk, (const __nv_bfloat16*)qw, (const __nv_bfloat16*)kw,
        (const float2*)cos_sin, seq, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_out, rstd_q, rstd_k, T,
        eps);
    return status();
  };
  if (head_dim == 128)
    return go(qk_norm_rope_fwd_kernel<128>, qk_block_threads<128>(nq + nk, QK_NB),
              qk_slot<128>(nq + nk, false));
  if (head_dim == 64)
    return go(qk_norm_rope_fwd_kernel<64>, qk_block_threads<64>(nq + nk, QK_NB),
              qk_slot<64>(nq + nk, false));
  return RP_E_INPUT;
}

RP_API int rp_qk_norm_rope_bwd(const void* dq, const void* dk, const void* qkv, int64_t ld,
                               int32_t nq, int32_t nk, int32_t head_dim, const void* qw,
                               const void* kw, const float* rstd_q, const float* rstd_k,
                               const float* cos_sin, int32_t seq, void* dqkv, int64_t ldd,
                               float* dqw, float* dkw, int32_t T, void* stream) {
  if (ld % 8 || ldd % 8 || T % 128 || T <= 0 || nq <= 0 || nk <= 0 || seq <= 0) return RP_E_INPUT;
  if (!qk_aligned(dq) || !qk_aligned(dk) || !qk_aligned(qkv) || !qk_aligned(cos_sin) ||
      !qk_aligned(qw) || !qk_aligned(kw) || !qk_aligned(dqkv))
    return RP_E_INPUT;
  const int rstd_bulk = nq % 4 == 0 && nk % 4 == 0 && qk_aligned(rstd_q) && qk_aligned(rstd_k);
  auto s = (cudaStream_t)stream;
  auto go = [&](auto kern, int bt, QkSlot L) -> int {
    const int smem = QK_STAGES_BWD * L.bytes + QK_STAGES_BWD * 8;
    if (!ensure_smem_t(kern, smem)) return RP_E_INPUT;
    kern<<<qk_wave_grid(kern, bt, smem, T), bt, smem, s>>>(
        (const __nv_bfloat16*)dq, (const __nv_bfloat16*)dk, (const __nv_bfloat16*)qkv, ld, nq, nk,
        (const __nv_bfloat16*)qw, (const __nv_bfloat16*)kw, rstd_q, rstd_k, (const float2*)cos_sin,
        seq, (__nv_bfloat16*)dqkv, ldd, dqw, dkw, T, rstd_bulk);
    return status();
  };
  if (head_dim == 128)
    return go(qk_norm_rope_bwd_kernel<128>, qk_block_threads<128>(nq + nk, QK_NB),
              qk_slot<128>(nq + nk, true));
  if (head_dim == 64)
    return go(qk_norm_rope_bwd_kernel<64>, qk_block_threads<64>(nq + nk, QK_NB),
              qk_slot<64>(nq + nk, true));
  return RP_E_INPUT;
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
