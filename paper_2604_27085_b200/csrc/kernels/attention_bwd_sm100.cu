// Causal GQA flash-attention BACKWARD on the 5th-gen tensor cores (sm_100a).
//
// Default (head_dim 128, even GQA group): (A4) below — ONE key-major kernel
// per (128-key block, query-head pair) forms dK, dV and dQ: S^T and dP^T per
// 64-query tile into TMEM, P^T / dS^T written back as bf16 A operands of
// dV += P^T dO and dK += dS^T Q, and dQ^T = K^T dS^T reduce-added (TMA, fp32,
// in L2) into a d-major accumulator — no S/dP recompute.
// Otherwise (head_dim 64 or odd GQA groups) two kernels:
//  (A/A2) dK/dV, key-major. CTA = 128 keys x 1 (A) or 2 (A2, ping-pong)
//      query heads; per 64-query tile S^T = K Q^T and dP^T = V dO^T (M128
//      N64) into double-buffered TMEM; softmax warps form P^T and dS^T;
//      dV += P^T dO and dK += dS^T Q accumulate in TMEM. GQA partials are
//      summed in fp32 (atomics), a cast kernel writes bf16.
//  (B3) dQ, query-major, Q and dO staged once into TMEM: S = Q K^T and
//      dP = dO V^T recomputed per 64-key tile, dQ += dS K.
#include <utility>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels/launch_util.h"
#include "kernels/sm100.cuh"
#include "rp/kernels.h"

namespace rp {
namespace {

using namespace sm100;
typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float ex2b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f;

// ====================================================================== (A) dK / dV
constexpr int A_BK = 128;                 // keys per CTA
constexpr int A_BQ = 64;                  // queries per tile
constexpr int SUB128 = 128 * 128;         // 128 rows x 64 bf16 (16 KB)
constexpr int SUB64 = 64 * 128;           // 64 rows x 64 bf16 (8 KB)
// Operand rings are 3 deep: a stage is released only after the gradient MMA
// of its tile, and with 2 stages the next S/dP MMA would wait a full TMA
// round trip behind that release on every tile.
constexpr int NST = 3;

template <int HD>
struct DkvSmem {
  static constexpr int NSUB = HD / 64;
  static constexpr int K = 0;
  static constexpr int V = K + NSUB * SUB128;
  static constexpr int Q0 = V + NSUB * SUB128;        // stage s: Q at Q0 + s*STAGE
  static constexpr int STAGE = 2 * NSUB * SUB64;      // Q + dO of one query tile
  static constexpr int DO_OFF = NSUB * SUB64;         // dO after Q inside a stage
  static constexpr int PS = Q0 + NST * STAGE;         // buffer b: P^T at PS + b*PS_BUF
  static constexpr int PS_BUF = 2 * (A_BK * A_BQ * 2);  // P^T + dS^T (16 KB each)
  static constexpr int LD = PS + 2 * PS_BUF;          // [NST][2][A_BQ] lse, delta
  static constexpr int BAR = LD + NST * 2 * A_BQ * 4;
  static constexpr int BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");
};

// CTA = (128-key block, query head): the causal work per key block shrinks
// linearly, so one CTA per (block, head) with the heaviest blocks first keeps
// the ~7 waves balanced; the G heads of a KV group reduce their dK/dV
// partials with 16-byte fp32 atomics into dk_acc / dv_acc.
template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkv_kernel(const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v,
                        const __grid_constant__ CUtensorMap tm_q,
                        const __grid_constant__ CUtensorMap tm_do, const float* __restrict__ lse,
                        const float* __restrict__ delta, float* __restrict__ dk_acc,
                        float* __restrict__ dv_acc, int T, int seq, int nq, int nk, float scale) {
  using L = DkvSmem<HD>;
  constexpr int NSUB = L::NSUB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;    // [NST]
  uint64_t* q_empty = bar + 4;   // [NST]
  uint64_t* sd_full = bar + 7;   // [2]
  uint64_t* sd_free = bar + 9;   // [2]
  uint64_t* ps_full = bar + 11;  // [2]
  uint64_t* ps_empty = bar + 13; // [2]
  uint64_t* acc_done = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kb = causal_block(blockIdx.y, T / A_BK, seq / A_BK, false), hq = blockIdx.x;
  const int kvh = hq / (nq / nk);
  const int k0 = kb * A_BK;
  const int s0 = (k0 / seq) * seq, s_end = s0 + seq;
  const int nqt = (s_end - k0) / A_BQ;  // query tiles at/after the diagonal
  const int iters = nqt;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    mbar_init(kv_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sd_full[i], 1);
      mbar_init(&sd_free[i], 8);
      mbar_init(&ps_full[i], 8);
      mbar_init(&ps_empty[i], 1);
    }
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S^T[b] at b*128 (64 cols), dP^T[b] at b*128+64, dV at 256, dK at 384
  const uint32_t TM_DV = 256, TM_DK = 384;

  if (warp == 0 && lane == 0) {
    mbar_arrive_expect_tx(kv_full, 2 * NSUB * SUB128);
    for (int sub = 0; sub < NSUB; ++sub) {
      tma_load_2d(sm + L::K + sub * SUB128, &tm_k, kv_full, kvh * HD + 64 * sub, k0);
      tma_load_2d(sm + L::V + sub * SUB128, &tm_v, kv_full, kvh * HD + 64 * sub, k0);
    }
    for (int it = 0; it < iters; ++it) {
      const int s = it % NST;
      mbar_wait(&q_empty[s], ((it / NST) & 1) ^ 1);
      const int qs = k0 + it * A_BQ;
      uint8_t* qd = sm + L::Q0 + s * L::STAGE;
      mbar_arrive_expect_tx(&q_full[s], L::STAGE + 2 * A_BQ * 4);
      for (int sub = 0; sub < NSUB; ++sub) {
        tma_load_2d(qd + sub * SUB64, &tm_q, &q_full[s], hq * HD + 64 * sub, qs);
        tma_load_2d(qd + L::DO_OFF + sub * SUB64, &tm_do, &q_full[s], hq * HD + 64 * sub, qs);
      }
      float* ld = reinterpret_cast<float*>(sm + L::LD) + s * 2 * A_BQ;
      bulk_load_1d(ld, lse + (long long)hq * T + qs, A_BQ * 4, &q_full[s]);
      bulk_load_1d(ld + A_BQ, delta + (long long)hq * T + qs, A_BQ * 4, &q_full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(A_BK, A_BQ, 0, 0);   // K-major x K-major
    constexpr uint32_t idesc_g = umma_idesc_bf16(A_BK, HD, 0, 1);     // K-major x MN-major
    const uint32_t k_addr = smem_u32(sm + L::K), v_addr = smem_u32(sm + L::V);
    auto issue_grads = [&](int it) {
      const int s = it % NST, b = it & 1;
      mbar_wait(&ps_full[b], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sm + L::Q0 + s * L::STAGE);
      const uint32_t do_addr = q_addr + L::DO_OFF;
      const uint32_t p_addr = smem_u32(sm + L::PS + b * L::PS_BUF);
      const uint32_t ds_addr = p_addr + A_BK * A_BQ * 2;
#pragma unroll
      for (int kk = 0; kk < A_BQ / 16; ++kk) {
        const uint64_t pa = umma_desc_sw128(p_addr + kk * 32, 16, 1024);
        const uint64_t da = umma_desc_sw128(ds_addr + kk * 32, 16, 1024);
        const uint64_t ob = umma_desc_sw128(do_addr + kk * 2048, SUB64, 1024);
        const uint64_t qb = umma_desc_sw128(q_addr + kk * 2048, SUB64, 1024);
        umma_f16(tmem + TM_DV, pa, ob, idesc_g, (it | kk) != 0);
        umma_f16(tmem + TM_DK, da, qb, idesc_g, (it | kk) != 0);
      }
      umma_commit(&ps_empty[b]);
      umma_commit(&q_empty[s]);
    };
    mbar_wait(kv_full, 0);
    for (int it = 0; it < iters; ++it) {
      const int s = it % NST, b = it & 1;
      mbar_wait(&q_full[s], (it / NST) & 1);
      if (it >= 2) mbar_wait(&sd_free[b], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t q_addr = smem_u32(sm + L::Q0 + s * L::STAGE);
      const uint32_t do_addr = q_addr + L::DO_OFF;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const uint32_t ko = (kk >> 2) * SUB128 + (kk & 3) * 32;
        const uint32_t qo = (kk >> 2) * SUB64 + (kk & 3) * 32;
        umma_f16(tmem + b * 128, umma_desc_sw128(k_addr + ko, 16, 1024),
                 umma_desc_sw128(q_addr + qo, 16, 1024), idesc_s, kk != 0);
        umma_f16(tmem + b * 128 + 64, umma_desc_sw128(v_addr + ko, 16, 1024),
                 umma_desc_sw128(do_addr + qo, 16, 1024), idesc_s, kk != 0);
      }
      umma_commit(&sd_full[b]);
      if (it >= 1) issue_grads(it - 1);
    }
    issue_grads(iters - 1);
    umma_commit(acc_done);
  } else if (warp >= 4) {
    // 8 softmax warps: lane quarter = warp % 4 (TMEM lanes = key rows), column
    // half = (warp - 4) / 4 (32 of the tile's 64 queries each)
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int r = quarter * 32 + lane;  // key row within the tile
    const int key = k0 + r;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    const float sl2 = scale * kLog2e;
    const int c0 = half * 32;
    for (int it = 0; it < iters; ++it) {
      const int b = it & 1;
      const int qs = k0 + it * A_BQ;
      // lse / delta of this tile arrive with its Q stage; the stage is only
      // refilled after this tile's gradient MMAs, i.e. after ps_full
      const int s = it % NST;
      const float* lse_t = reinterpret_cast<const float*>(sm + L::LD) + s * 2 * A_BQ;
      const float* del_t = lse_t + A_BQ;
      mbar_wait(&q_full[s], (it / NST) & 1);  // lse/delta visibility (already complete)
      mbar_wait(&sd_full[b], (it >> 1) & 1);
      tc_fence_after();
      uint32_t sv[32], dpv[32];
      tmem_ld_32x32b_x32(lane_base + b * 128 + c0, sv);
      tmem_ld_32x32b_x32(lane_base + b * 128 + 64 + c0, dpv);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sd_free[b]);
      uint32_t pk[16], dk2[16];
      const bool diag = qs + A_BQ > k0 && qs < k0 + A_BK;  // tile crosses this key block
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const int c = c0 + i;
        float p0 = ex2b(fmaf(__uint_as_float(sv[i]), sl2, -lse_t[c] * kLog2e));
        float p1 = ex2b(fmaf(__uint_as_float(sv[i + 1]), sl2, -lse_t[c + 1] * kLog2e));
        if (diag) {
          if (qs + c < key) p0 = 0.f;
          if (qs + c + 1 < key) p1 = 0.f;
        }
        const float d0 = p0 * (__uint_as_float(dpv[i]) - del_t[c]);
        const float d1 = p1 * (__uint_as_float(dpv[i + 1]) - del_t[c + 1]);
        pk[i / 2] = pack_bf16x2(p0, p1);
        dk2[i / 2] = pack_bf16x2(d0, d1);
      }
      if (it >= 2) {
        mbar_wait(&ps_empty[b], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
      }
      uint8_t* prow = sm + L::PS + b * L::PS_BUF + (r >> 3) * 1024 + (r & 7) * 128;
      uint8_t* drow = prow + A_BK * A_BQ * 2;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int off = ((half * 4 + q4) ^ (r & 7)) << 4;
        *reinterpret_cast<uint4*>(prow + off) =
            make_uint4(pk[q4 * 4], pk[q4 * 4 + 1], pk[q4 * 4 + 2], pk[q4 * 4 + 3]);
        *reinterpret_cast<uint4*>(drow + off) =
            make_uint4(dk2[q4 * 4], dk2[q4 * 4 + 1], dk2[q4 * 4 + 2], dk2[q4 * 4 + 3]);
      }
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps_full[b]);
    }
    // epilogue: dK (scaled) and dV rows, reduced over the G heads in fp32
    mbar_wait(acc_done, 0);
    tc_fence_after();
    float* dkr = dk_acc + (long long)key * nk * HD + (long long)kvh * HD;
    float* dvr = dv_acc + (long long)key * nk * HD + (long long)kvh * HD;
#pragma unroll 1
    for (int c = half * (HD / 2); c < (half + 1) * (HD / 2); c += 32) {
      uint32_t a[32], v[32];
      tmem_ld_32x32b_x32(lane_base + TM_DK + c, a);
      tmem_ld_32x32b_x32(lane_base + TM_DV + c, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        atomicAdd(reinterpret_cast<float4*>(dkr + c + i),
                  make_float4(__uint_as_float(a[i]) * scale, __uint_as_float(a[i + 1]) * scale,
                              __uint_as_float(a[i + 2]) * scale, __uint_as_float(a[i + 3]) * scale));
        atomicAdd(reinterpret_cast<float4*>(dvr + c + i),
                  make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                              __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3])));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================ (A2) dK / dV, ping-pong
// CTA = 128 keys x TWO query heads (ha, ha+1) of one KV group. Both heads'
// dV/dK land in the SAME TMEM accumulators (dV_kv = sum_h P_h^T dO_h), and
// the two softmax warpgroups alternate with the tensor core, which runs
//   S/dP_a(j) | grads_b(j-1) | S/dP_b(j) | grads_a(j) | S/dP_a(j+1) | ...
// so each warpgroup's P^T/dS^T work hides behind ~1024 cycles of the other
// head's MMAs. P^T and dS^T (bf16) are written back into the TMEM columns of
// the S^T / dP^T they came from and feed the dV / dK MMAs as TMEM A operands
// (tcgen05.mma ... [a_tmem]); the shared memory this saves deepens the
// (Q, dO, lse, delta) ring to 4 slots, consumed in the order (j, a), (j, b),
// (j+1, a), ... so each tile's TMA load has ~2 K cycles of lead.
constexpr int A2_THREADS = 384;
constexpr int A2_NST = 4;

template <int HD>
struct Dkv2Smem {
  static constexpr int NSUB = HD / 64;
  static constexpr int K = 0;
  static constexpr int V = K + NSUB * SUB128;
  static constexpr int R0 = V + NSUB * SUB128;        // ring slot s at R0 + s*STAGE
  static constexpr int STAGE = 2 * NSUB * SUB64;      // Q + dO of one (tile, head)
  static constexpr int DO_OFF = NSUB * SUB64;
  static constexpr int LD = R0 + A2_NST * STAGE;      // [A2_NST][2][A_BQ] lse, delta
  static constexpr int BAR = LD + A2_NST * 2 * A_BQ * 4;
  static constexpr int BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");
};

template <int HD>
__global__ void __launch_bounds__(A2_THREADS, 1)
    attn_bwd_dkv_pp_kernel(const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v,
                           const __grid_constant__ CUtensorMap tm_q,
                           const __grid_constant__ CUtensorMap tm_do,
                           const float* __restrict__ lse, const float* __restrict__ delta,
                           float* __restrict__ dk_acc, float* __restrict__ dv_acc, int T, int seq,
                           int nq, int nk, float scale) {
  using L = Dkv2Smem<HD>;
  constexpr int NSUB = L::NSUB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* st_full = bar + 1;            // [A2_NST]
  uint64_t* st_empty = bar + 1 + A2_NST;  // [A2_NST]
  uint64_t* sd_full = bar + 1 + 2 * A2_NST;  // [2] per head
  uint64_t* ps_full = sd_full + 2;           // [2]
  uint64_t* acc_done = ps_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kb = causal_block(blockIdx.y, T / A_BK, seq / A_BK, false), ha = 2 * (int)blockIdx.x;
  const int kvh = ha / (nq / nk);
  const int k0 = kb * A_BK;
  const int s0 = (k0 / seq) * seq, s_end = s0 + seq;
  const int nqt = (s_end - k0) / A_BQ;  // query tiles at/after the diagonal

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    mbar_init(kv_full, 1);
    for (int i = 0; i < A2_NST; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sd_full[i], 1);
      mbar_init(&ps_full[i], 4);
    }
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: head w: S^T at w*128 (64 cols), dP^T at w*128 + 64; after the
  // softmax pass P^T (bf16 pairs) occupies w*128 + [0, 32) and dS^T
  // w*128 + 64 + [0, 32). dV at 256, dK at 384.
  const uint32_t TM_DV = 256, TM_DK = 384;

  if (warp == 0 && lane == 0) {
    mbar_arrive_expect_tx(kv_full, 2 * NSUB * SUB128);
    for (int sub = 0; sub < NSUB; ++sub) {
      tma_load_2d(sm + L::K + sub * SUB128, &tm_k, kv_full, kvh * HD + 64 * sub, k0);
      tma_load_2d(sm + L::V + sub * SUB128, &tm_v, kv_full, kvh * HD + 64 * sub, k0);
    }
    for (int idx = 0; idx < 2 * nqt; ++idx) {
      const int s = idx % A2_NST, w = idx & 1, hq = ha + w;
      mbar_wait(&st_empty[s], ((idx / A2_NST) & 1) ^ 1);
      const int qs = k0 + (idx >> 1) * A_BQ;
      uint8_t* qd = sm + L::R0 + s * L::STAGE;
      mbar_arrive_expect_tx(&st_full[s], L::STAGE + 2 * A_BQ * 4);
      for (int sub = 0; sub < NSUB; ++sub) {
        tma_load_2d(qd + sub * SUB64, &tm_q, &st_full[s], hq * HD + 64 * sub, qs);
        tma_load_2d(qd + L::DO_OFF + sub * SUB64, &tm_do, &st_full[s], hq * HD + 64 * sub, qs);
      }
      float* ld = reinterpret_cast<float*>(sm + L::LD) + s * 2 * A_BQ;
      bulk_load_1d(ld, lse + (long long)hq * T + qs, A_BQ * 4, &st_full[s]);
      bulk_load_1d(ld + A_BQ, delta + (long long)hq * T + qs, A_BQ * 4, &st_full[s]);
    }
  } else if (warp == 1) {  // whole warp: uniform descriptors, elected issue
    constexpr uint32_t idesc_s = umma_idesc_bf16(A_BK, A_BQ, 0, 0);   // K-major x K-major
    constexpr uint32_t idesc_g = umma_idesc_bf16(A_BK, HD, 0, 1);     // K-major x MN-major
    const uint32_t k_addr = smem_u32(sm + L::K), v_addr = smem_u32(sm + L::V);
    auto stage = [&](int idx) { return smem_u32(sm + L::R0 + (idx % A2_NST) * L::STAGE); };
    auto issue_sdp = [&](int j, int w) {
      const int idx = 2 * j + w;
      mbar_wait(&st_full[idx % A2_NST], (idx / A2_NST) & 1);
      tc_fence_after();
      const uint32_t q_addr = stage(idx), do_addr = q_addr + L::DO_OFF;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * SUB128 + (kk & 3) * 32;
          const uint32_t qo = (kk >> 2) * SUB64 + (kk & 3) * 32;
          umma_f16(tmem + w * 128, umma_desc_sw128(k_addr + ko, 16, 1024),
                   umma_desc_sw128(q_addr + qo, 16, 1024), idesc_s, kk != 0);
          umma_f16(tmem + w * 128 + 64, umma_desc_sw128(v_addr + ko, 16, 1024),
                   umma_desc_sw128(do_addr + qo, 16, 1024), idesc_s, kk != 0);
        }
        umma_commit(&sd_full[w]);
      }
      __syncwarp();
    };
    auto issue_grads = [&](int j, int w) {
      const int idx = 2 * j + w;
      mbar_wait(&ps_full[w], j & 1);
      tc_fence_after();
      const uint32_t q_addr = stage(idx), do_addr = q_addr + L::DO_OFF;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < A_BQ / 16; ++kk) {
          const uint64_t ob = umma_desc_sw128(do_addr + kk * 2048, SUB64, 1024);
          const uint64_t qb = umma_desc_sw128(q_addr + kk * 2048, SUB64, 1024);
          umma_f16_ts(tmem + TM_DV, tmem + w * 128 + kk * 8, ob, idesc_g, (idx | kk) != 0);
          umma_f16_ts(tmem + TM_DK, tmem + w * 128 + 64 + kk * 8, qb, idesc_g, (idx | kk) != 0);
        }
        umma_commit(&st_empty[idx % A2_NST]);
      }
      __syncwarp();
    };
    mbar_wait(kv_full, 0);
    issue_sdp(0, 0);
    issue_sdp(0, 1);
    for (int j = 0; j < nqt; ++j) {
      issue_grads(j, 0);
      if (j + 1 < nqt) issue_sdp(j + 1, 0);  // in-order after grads_a(j) read P^T_a
      issue_grads(j, 1);
      if (j + 1 < nqt) issue_sdp(j + 1, 1);
    }
    if (elect_one()) umma_commit(acc_done);
    __syncwarp();
  } else if (warp >= 4) {
    // two softmax warpgroups: w = head slot, thread = key row
    const int w = (warp - 4) >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int key = k0 + r;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    const float sl2 = scale * kLog2e;
    for (int j = 0; j < nqt; ++j) {
      const int idx = 2 * j + w, s = idx % A2_NST;
      const int qs = k0 + j * A_BQ;
      const float* lse_t = reinterpret_cast<const float*>(sm + L::LD) + s * 2 * A_BQ;
      const float* del_t = lse_t + A_BQ;
      mbar_wait(&st_full[s], (idx / A2_NST) & 1);  // lse/delta visibility (already complete)
      mbar_wait(&sd_full[w], j & 1);
      tc_fence_after();
      const bool diag = qs < k0 + A_BK;  // tile overlaps this key block's diagonal
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t sv[32], dpv[32], pk[16], dk2[16];
        tmem_ld_32x32b_x32(lane_base + w * 128 + half * 32, sv);
        tmem_ld_32x32b_x32(lane_base + w * 128 + 64 + half * 32, dpv);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const int c = half * 32 + i;
          float p0 = ex2b(fmaf(__uint_as_float(sv[i]), sl2, -lse_t[c] * kLog2e));
          float p1 = ex2b(fmaf(__uint_as_float(sv[i + 1]), sl2, -lse_t[c + 1] * kLog2e));
          if (diag) {
            if (qs + c < key) p0 = 0.f;
            if (qs + c + 1 < key) p1 = 0.f;
          }
          const float d0 = p0 * (__uint_as_float(dpv[i]) - del_t[c]);
          const float d1 = p1 * (__uint_as_float(dpv[i + 1]) - del_t[c + 1]);
          pk[i / 2] = pack_bf16x2(p0, p1);
          dk2[i / 2] = pack_bf16x2(d0, d1);
        }
        // bf16 pairs back over columns this thread has already read
        tmem_st_32x32b_x16(lane_base + w * 128 + half * 16, pk);
        tmem_st_32x32b_x16(lane_base + w * 128 + 64 + half * 16, dk2);
      }
      tmem_st_wait_all();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps_full[w]);
    }
    // epilogue: warpgroup a -> dK (scaled), warpgroup b -> dV; fp32 atomics
    // reduce the G/2 head pairs of the KV group
    mbar_wait(acc_done, 0);
    tc_fence_after();
    float* dst = (w == 0 ? dk_acc : dv_acc) + (long long)key * nk * HD + (long long)kvh * HD;
    const uint32_t col = w == 0 ? TM_DK : TM_DV;
    const float f = w == 0 ? scale : 1.f;
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t a[32];
      tmem_ld_32x32b_x32(lane_base + col + c, a);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        atomicAdd(reinterpret_cast<float4*>(dst + c + i),
                  make_float4(__uint_as_float(a[i]) * f, __uint_as_float(a[i + 1]) * f,
                              __uint_as_float(a[i + 2]) * f, __uint_as_float(a[i + 3]) * f));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================ (A4) dK / dV / dQ in one kernel
// The ping-pong dK/dV kernel (A2) plus dQ: after the softmax pass P^T and
// dS^T (bf16) sit in the first 64 TMEM columns of the head's S^T|dP^T block,
// so the last 64 hold dQ^T = K^T dS^T (M = head_dim, N = 64 queries; K^T is
// the MN-major view of the resident K tile, dS^T a bf16 copy in shared
// memory). This removes the dQ kernel's recompute of S and dP (2 of its 3
// MMA units) and its exp pass.
//
// Four warpgroups (512 threads, registers rebalanced with setmaxnreg):
//   WG0  w0 TMA producer, w1 MMA issuer (w2, w3 idle)             56 regs
//   WG1  softmax of head a, WG2 softmax of head b (thread = key)  184 regs
//   WG3  dQ drain for both heads (thread = head-dim lane): TMEM ->
//        registers -> swizzled staging -> TMA reduce-add into a d-major
//        fp32 dQ^T accumulator in L2 (cp.reduce.async.bulk .add.f32)    88 regs
// The softmax warpgroups never wait for dQ: their loop is S^T/dP^T in,
// P^T/dS^T out. Tensor-core order per (query tile j, head w):
//   dQ^T(j,w) | dV,dK(j,w) | S^T(j+1,w) | [dQ^T(j,w) drained] dP^T(j+1,w)
// so the drain of dQ^T (which shares TMEM columns with dP^T) hides behind
// ~900 cycles of MMAs instead of stalling the tensor pipe.
constexpr int A4_NST = 3;
constexpr int A4_THREADS = 512;


template <int HD>
struct Dkv4Smem {
  static constexpr int NSUB = HD / 64;
  static constexpr int K = 0;
  static constexpr int V = K + NSUB * SUB128;
  static constexpr int R0 = V + NSUB * SUB128;     // ring slot s at R0 + s*STAGE
  static constexpr int STAGE = 2 * NSUB * SUB64;   // Q + dO of one (tile, head)
  static constexpr int DO_OFF = NSUB * SUB64;
  static constexpr int DST = R0 + A4_NST * STAGE;  // [2] dS^T [128 keys][64 q] bf16, SW128
  static constexpr int STG = DST + 2 * A_BK * A_BQ * 2;  // [4 drain warps][2 halves] 4 KB
  static constexpr int LD = STG + 8 * 4096;        // [A4_NST][2][A_BQ] -lse*log2e, delta
  static constexpr int BAR = LD + A4_NST * 2 * A_BQ * 4;
  static constexpr int BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");
};

__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src,
                                                  int32_t c0, int32_t c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::
          "l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit_grp() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_done_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// GQA reduction of dK/dV over the G/2 head pairs of a KV group (CL):
//   0: fp32 atomics into dk_acc / dv_acc (+ a cast kernel), any G
//   1: G = 2, one CTA per group: bf16 straight from TMEM into dk / dv
//   2: G = 4, the two CTAs of a group form a cluster: rank 1 ships its fp32
//      dK/dV rows into rank 0's (then idle) shared memory over DSMEM, rank 0
//      adds them to its own and writes bf16 — no atomics, memset or cast
// `nlse2` = -lse * log2(e) per (head, query), written by delta_kernel.
template <int HD, int CL>
__global__ void __launch_bounds__(A4_THREADS, 1)
    attn_bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v,
                          const __grid_constant__ CUtensorMap tm_q,
                          const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_dq,
                          const float* __restrict__ nlse2, const float* __restrict__ delta,
                          float* __restrict__ dk_acc, float* __restrict__ dv_acc,
                          bf16* __restrict__ dk, long long lddk, bf16* __restrict__ dv,
                          long long lddv, int T, int seq, int nq, int nk, float scale) {
  using L = Dkv4Smem<HD>;
  constexpr int NSUB = L::NSUB;
  constexpr int NS = A4_NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* kv_full = bar + 0;
  uint64_t* st_full = bar + 1;             // [NS]
  uint64_t* st_empty = bar + 1 + NS;       // [NS]
  uint64_t* sd_full = bar + 1 + 2 * NS;    // [2] per head
  uint64_t* ps_full = sd_full + 2;         // [2]
  uint64_t* dq_full = ps_full + 2;         // [2]
  uint64_t* dq_free = dq_full + 2;         // [2]
  uint64_t* acc_done = dq_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int kb = causal_block(blockIdx.y, T / A_BK, seq / A_BK, false), ha = 2 * (int)blockIdx.x;
  const int kvh = ha / (nq / nk);
  const int k0 = kb * A_BK;
  const int s0 = (k0 / seq) * seq, s_end = s0 + seq;
  const int nqt = (s_end - k0) / A_BQ;  // query tiles at/after the diagonal

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    mbar_init(kv_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sd_full[i], 1);
      mbar_init(&ps_full[i], 4);
      mbar_init(&dq_full[i], 1);
      mbar_init(&dq_free[i], 4);
    }
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM per head w: S^T at w*128 (64 cols), dP^T at w*128 + 64; after the
  // softmax pass P^T (bf16 pairs) at w*128 + [0, 32), dS^T at w*128 + [32, 64)
  // and dQ^T (fp32, lane = head dim) at w*128 + [64, 128). dV at 256, dK at 384.
  const uint32_t TM_DV = 256, TM_DK = 384;
  const bool softmax_wg = warp >= 4 && warp < 12;

  // cluster-wide barrier (CL == 2 epilogue); every thread of both CTAs takes part
  auto cluster_sync = [] {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
  };

  if (warp < 4) {
  setmaxnreg_dec<112>();
  if (warp == 0 && lane == 0) {
    mbar_arrive_expect_tx(kv_full, 2 * NSUB * SUB128);
    for (int sub = 0; sub < NSUB; ++sub) {
      tma_load_2d(sm + L::K + sub * SUB128, &tm_k, kv_full, kvh * HD + 64 * sub, k0);
      tma_load_2d(sm + L::V + sub * SUB128, &tm_v, kv_full, kvh * HD + 64 * sub, k0);
    }
    for (int idx = 0; idx < 2 * nqt; ++idx) {
      const int s = idx % NS, w = idx & 1, hq = ha + w;
      mbar_wait(&st_empty[s], ((idx / NS) & 1) ^ 1);
      const int qs = k0 + (idx >> 1) * A_BQ;
      uint8_t* qd = sm + L::R0 + s * L::STAGE;
      mbar_arrive_expect_tx(&st_full[s], L::STAGE + 2 * A_BQ * 4);
      for (int sub = 0; sub < NSUB; ++sub) {
        tma_load_2d(qd + sub * SUB64, &tm_q, &st_full[s], hq * HD + 64 * sub, qs);
        tma_load_2d(qd + L::DO_OFF + sub * SUB64, &tm_do, &st_full[s], hq * HD + 64 * sub, qs);
      }
      float* ld = reinterpret_cast<float*>(sm + L::LD) + s * 2 * A_BQ;
      bulk_load_1d(ld, nlse2 + (long long)hq * T + qs, A_BQ * 4, &st_full[s]);
      bulk_load_1d(ld + A_BQ, delta + (long long)hq * T + qs, A_BQ * 4, &st_full[s]);
    }
  } else if (warp == 1) {  // whole warp: uniform descriptors, elected issue
    constexpr uint32_t idesc_s = umma_idesc_bf16(A_BK, A_BQ, 0, 0);  // K-major x K-major
    constexpr uint32_t idesc_g = umma_idesc_bf16(A_BK, HD, 0, 1);    // TMEM A x MN-major
    constexpr uint32_t idesc_q = umma_idesc_bf16(HD, A_BQ, 1, 1);    // MN-major x MN-major
    const uint32_t k_addr = smem_u32(sm + L::K), v_addr = smem_u32(sm + L::V);
    auto stage = [&](int idx) { return smem_u32(sm + L::R0 + (idx % NS) * L::STAGE); };
    // S^T = K Q^T into w*128 (ops 0) or dP^T = V dO^T into w*128 + 64 (ops 1)
    auto issue_sd = [&](int idx, int w, int which) {
      const uint32_t b_addr = stage(idx) + (which ? L::DO_OFF : 0);
      const uint32_t a_addr = which ? v_addr : k_addr;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * SUB128 + (kk & 3) * 32;
          const uint32_t qo = (kk >> 2) * SUB64 + (kk & 3) * 32;
          umma_f16(tmem + w * 128 + which * 64, umma_desc_sw128(a_addr + ko, 16, 1024),
                   umma_desc_sw128(b_addr + qo, 16, 1024), idesc_s, kk != 0);
        }
      }
      __syncwarp();
    };
    auto wait_stage = [&](int idx) {
      mbar_wait(&st_full[idx % NS], (idx / NS) & 1);
      tc_fence_after();
    };
    mbar_wait(kv_full, 0);
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      wait_stage(w);
      issue_sd(w, w, 0);
      issue_sd(w, w, 1);
      if (elect_one()) umma_commit(&sd_full[w]);
      __syncwarp();
    }
    for (int j = 0; j < nqt; ++j) {
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int idx = 2 * j + w;
        mbar_wait(&ps_full[w], j & 1);
        tc_fence_after();
        const uint32_t q_addr = stage(idx), do_addr = q_addr + L::DO_OFF;
        const uint32_t ds_addr = smem_u32(sm + L::DST + w * (A_BK * A_BQ * 2));
        if (elect_one()) {
          // dQ^T = K^T dS^T over the 128 keys of this block (first, so its
          // drain overlaps the dV/dK and next S^T MMAs)
#pragma unroll
          for (int kk = 0; kk < A_BK / 16; ++kk)
            umma_f16(tmem + w * 128 + 64, umma_desc_sw128(k_addr + kk * 2048, SUB128, 1024),
                     umma_desc_sw128(ds_addr + kk * 2048, 8192, 1024), idesc_q, kk != 0);
          umma_commit(&dq_full[w]);
#pragma unroll
          for (int kk = 0; kk < A_BQ / 16; ++kk) {
            const uint64_t ob = umma_desc_sw128(do_addr + kk * 2048, SUB64, 1024);
            const uint64_t qb = umma_desc_sw128(q_addr + kk * 2048, SUB64, 1024);
            umma_f16_ts(tmem + TM_DV, tmem + w * 128 + kk * 8, ob, idesc_g, (idx | kk) != 0);
            umma_f16_ts(tmem + TM_DK, tmem + w * 128 + 32 + kk * 8, qb, idesc_g, (idx | kk) != 0);
          }
          umma_commit(&st_empty[idx % NS]);
        }
        __syncwarp();
        if (j + 1 < nqt) {
          wait_stage(idx + 2);
          issue_sd(idx + 2, w, 0);          // S^T(j+1) over P^T/dS^T(j): in order
          mbar_wait(&dq_free[w], j & 1);    // dQ^T(j) drained from the dP^T columns
          tc_fence_after();
          issue_sd(idx + 2, w, 1);
          if (elect_one()) umma_commit(&sd_full[w]);
          __syncwarp();
        }
      }
    }
    if (elect_one()) umma_commit(acc_done);
    __syncwarp();
  }
  __syncwarp();
  if (CL == 2) {  // partner CTA's epilogue exchange (see the softmax branch)
    cluster_sync();
    cluster_sync();
  }
  } else if (softmax_wg) {
    setmaxnreg_inc<160>();
    // softmax warpgroup w (head ha + w), thread = key row
    const int w = (warp - 4) >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int key = k0 + r;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    const float2 sl2 = make_float2(scale * kLog2e, scale * kLog2e);
    uint8_t* dst = sm + L::DST + w * (A_BK * A_BQ * 2);  // this head's dS^T
    for (int j = 0; j < nqt; ++j) {
      const int idx = 2 * j + w, s = idx % NS;
      const int jq = j * A_BQ;  // query offset of the tile from k0
      const float4* nl4 = reinterpret_cast<const float4*>(sm + L::LD) + s * 2 * A_BQ / 4;
      const float4* dl4 = nl4 + A_BQ / 4;
      mbar_wait(&st_full[s], (idx / NS) & 1);  // lse/delta visibility (already complete)
      mbar_wait(&sd_full[w], j & 1);
      tc_fence_after();
      const bool diag = jq < A_BK;  // tile overlaps this key block's diagonal
      uint32_t pk[32], dk2[32];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t sv[32], dpv[32];
        tmem_ld_32x32b_x32(lane_base + w * 128 + half * 32, sv);
        tmem_ld_32x32b_x32(lane_base + w * 128 + 64 + half * 32, dpv);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const int c = half * 32 + i;
          const float4 nl = nl4[c / 4], dl = dl4[c / 4];
          const float2 a0 = __ffma2_rn(make_float2(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])),
                                       sl2, make_float2(nl.x, nl.y));
          const float2 a1 = __ffma2_rn(make_float2(__uint_as_float(sv[i + 2]), __uint_as_float(sv[i + 3])),
                                       sl2, make_float2(nl.z, nl.w));
          float2 p0 = make_float2(ex2b(a0.x), ex2b(a0.y));
          float2 p1 = make_float2(ex2b(a1.x), ex2b(a1.y));
          if (diag) {  // key r sees queries jq + c >= r only
            if (jq + c < r) p0.x = 0.f;
            if (jq + c + 1 < r) p0.y = 0.f;
            if (jq + c + 2 < r) p1.x = 0.f;
            if (jq + c + 3 < r) p1.y = 0.f;
          }
          const float2 d0 = __fmul2_rn(p0, __fadd2_rn(make_float2(__uint_as_float(dpv[i]),
                                                                  __uint_as_float(dpv[i + 1])),
                                                      make_float2(-dl.x, -dl.y)));
          const float2 d1 = __fmul2_rn(p1, __fadd2_rn(make_float2(__uint_as_float(dpv[i + 2]),
                                                                  __uint_as_float(dpv[i + 3])),
                                                      make_float2(-dl.z, -dl.w)));
          pk[c / 2] = pack_bf16x2(p0.x, p0.y);
          pk[c / 2 + 1] = pack_bf16x2(p1.x, p1.y);
          dk2[c / 2] = pack_bf16x2(d0.x, d0.y);
          dk2[c / 2 + 1] = pack_bf16x2(d1.x, d1.y);
        }
      }
      // every S^T / dP^T column of this thread has been read: P^T -> [0, 32),
      // dS^T -> [32, 64)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t a[16], b[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          a[i] = pk[h * 16 + i];
          b[i] = dk2[h * 16 + i];
        }
        tmem_st_32x32b_x16(lane_base + w * 128 + h * 16, a);
        tmem_st_32x32b_x16(lane_base + w * 128 + 32 + h * 16, b);
      }
      // dS^T (bf16) into shared memory for dQ^T = K^T dS^T: row = key (128 B),
      // SWIZZLE_128B; dQ^T(j-1) read it before S^T/dP^T(j) were committed
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(dst + r * 128 + ((c ^ (r & 7)) << 4)) =
            make_uint4(dk2[4 * c], dk2[4 * c + 1], dk2[4 * c + 2], dk2[4 * c + 3]);
      fence_proxy_async();
      tmem_st_wait_all();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ps_full[w]);
    }
    // epilogue: warpgroup a -> dK (scaled), warpgroup b -> dV
    mbar_wait(acc_done, 0);
    tc_fence_after();
    if (CL == 0) {  // fp32 atomics reduce the G/2 head pairs of the KV group
      float* dst_acc = (w == 0 ? dk_acc : dv_acc) + (long long)key * nk * HD + (long long)kvh * HD;
      const uint32_t col = w == 0 ? TM_DK : TM_DV;
      const float f = w == 0 ? scale : 1.f;
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t a[32];
        tmem_ld_32x32b_x32(lane_base + col + c, a);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          atomicAdd(reinterpret_cast<float4*>(dst_acc + c + i),
                    make_float4(__uint_as_float(a[i]) * f, __uint_as_float(a[i + 1]) * f,
                                __uint_as_float(a[i + 2]) * f, __uint_as_float(a[i + 3]) * f));
      }
    }
    if (CL >= 1) {
    // dK / dV rows of this key block: thread = key row, HD fp32 per row; the
    // partner's rows arrive in this CTA's ring + dS^T region (2 x 128 x HD fp32,
    // 16-byte chunks XOR-swizzled by row so 32 rows hit 32 different banks)
    uint32_t rank = 0;
    if (CL == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t col = w == 0 ? TM_DK : TM_DV;
    constexpr int CH = HD / 4;  // 16-byte chunks per row
    float* xbuf = reinterpret_cast<float*>(sm + L::R0) + (size_t)w * A_BK * HD + (size_t)r * HD;
    auto chunk = [&](int c4) { return ((c4 ^ (r & (CH - 1))) * 4); };
    if (CL == 2) {
      cluster_sync();  // rank 0's ring / dS^T shared memory is free
      if (rank == 1) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(xbuf)));
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t a[32];
          tmem_ld_32x32b_x32(lane_base + col + c, a);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                             remote + chunk((c + i) / 4) * 4),
                         "f"(__uint_as_float(a[i])), "f"(__uint_as_float(a[i + 1])),
                         "f"(__uint_as_float(a[i + 2])), "f"(__uint_as_float(a[i + 3]))
                         : "memory");
        }
      }
      cluster_sync();
    }
    if (rank == 0) {
      bf16* dst = (w == 0 ? dk + (long long)key * lddk : dv + (long long)key * lddv) +
                  (long long)kvh * HD;
      const float f = w == 0 ? scale : 1.f;
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t a[32];
        tmem_ld_32x32b_x32(lane_base + col + c, a);
        tmem_ld_wait();
        float o[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(a[i]);
        if (CL == 2) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b = *reinterpret_cast<const float4*>(xbuf + chunk((c + i) / 4));
            o[i] += b.x;
            o[i + 1] += b.y;
            o[i + 2] += b.z;
            o[i + 3] += b.w;
          }
        }
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(dst + c + i) =
              make_uint4(pack_bf16x2(o[i] * f, o[i + 1] * f), pack_bf16x2(o[i + 2] * f, o[i + 3] * f),
                         pack_bf16x2(o[i + 4] * f, o[i + 5] * f), pack_bf16x2(o[i + 6] * f, o[i + 7] * f));
      }
    }
  }
  } else {
    setmaxnreg_dec<80>();
    // dQ drain warpgroup, thread = head-dim lane d = quarter*32 + lane; per
    // (tile, head): TMEM -> registers, release the columns, stage two
    // [32 dims][32 queries] fp32 blocks (one SWIZZLE_128B row per dim) and
    // reduce-add them into the d-major dQ^T accumulator
    const int quarter = warp & 3;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    uint8_t* stg = sm + L::STG + quarter * 8192;
    for (int idx = 0; idx < 2 * nqt; ++idx) {
      const int w = idx & 1, j = idx >> 1;
      const int qs = k0 + j * A_BQ;
      mbar_wait(&dq_full[w], j & 1);
      tc_fence_after();
      uint32_t q0v[32], q1v[32];
      tmem_ld_32x32b_x32(lane_base + w * 128 + 64, q0v);
      tmem_ld_32x32b_x32(lane_base + w * 128 + 96, q1v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dq_free[w]);
      if (lane == 0) bulk_wait_read_all();  // this warp's previous reduces left the staging
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        *reinterpret_cast<uint4*>(stg + lane * 128 + ((k ^ (lane & 7)) << 4)) =
            make_uint4(q0v[4 * k], q0v[4 * k + 1], q0v[4 * k + 2], q0v[4 * k + 3]);
        *reinterpret_cast<uint4*>(stg + 4096 + lane * 128 + ((k ^ (lane & 7)) << 4)) =
            make_uint4(q1v[4 * k], q1v[4 * k + 1], q1v[4 * k + 2], q1v[4 * k + 3]);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        const int hq = ha + w;
        tma_reduce_add_2d(&tm_dq, stg, qs, hq * HD + quarter * 32);
        tma_reduce_add_2d(&tm_dq, stg + 4096, qs + 32, hq * HD + quarter * 32);
        bulk_commit_grp();
      }
    }
    if (lane == 0) bulk_wait_done_all();
    __syncwarp();
    if (CL == 2) {
      cluster_sync();
      cluster_sync();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ======================================================================== (B) dQ
// query-major dQ kernel of the two-kernel path (head_dim 64 / odd GQA groups)
constexpr int B_Q = 128;  // queries per CTA
constexpr int B_K = 64;   // keys per tile

// ============================================================ (B3) dQ, operands in TMEM
// CTA = 128 queries x 1 head. Q and dO are staged ONCE into TMEM (bf16 pairs,
// row = lane) and are the A operands of S = Q K^T and dP = dO V^T, so the
// shared-memory port only carries the K/V tiles (B operands); S/dP are
// double-buffered so the tensor core computes S/dP(j+1) and dQ(j) while 8
// softmax warps (2 per lane quarter, one 32-key half each) turn tile j into
// dS, written back as bf16 pairs into the columns of S they read (half 0 ->
// cols [0,16), half 1 -> [32,48)), the A operand of dQ += dS K.
constexpr int B3_NST = 5;

template <int HD>
struct Dq3Smem {
  static constexpr int NSUB = HD / 64;
  static constexpr int STAGE = 2 * NSUB * SUB64;  // K_j + V_j (64 keys)
  static constexpr int BAR = B3_NST * STAGE;
  static constexpr int BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");
};

template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq3_kernel(const bf16* __restrict__ q, long long ldq, const bf16* __restrict__ dout,
                        long long lddo, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const float* __restrict__ lse,
                        const float* __restrict__ delta, bf16* __restrict__ dq, long long lddq,
                        int T, int seq, int nq, int nk, float scale) {
  using L = Dq3Smem<HD>;
  constexpr int NSUB = L::NSUB;
  constexpr uint32_t TQ = 0, TDO = HD / 2, TS = HD, TDQ = HD + 256;  // TMEM columns
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_ready = bar + 0;
  uint64_t* kv_full = bar + 1;            // [B3_NST]
  uint64_t* kv_empty = bar + 1 + B3_NST;  // [B3_NST]
  uint64_t* sd_full = kv_empty + B3_NST;  // [2]
  uint64_t* ds_full = sd_full + 2;        // [2]
  uint64_t* dq_done = ds_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qblocks = T / B_Q;
  const int qb = causal_block(blockIdx.y, qblocks, seq / B_Q, true);
  const int h = blockIdx.x, kvh = h / (nq / nk);
  const int q0 = qb * B_Q;
  const int s0 = (q0 / seq) * seq;
  const int ntiles = (q0 - s0) / B_K + B_Q / B_K;  // keys [s0, q0 + 128)

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    mbar_init(q_ready, 8);
    for (int i = 0; i < B3_NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sd_full[i], 1);
      mbar_init(&ds_full[i], 8);
    }
    mbar_init(dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    for (int j = 0; j < ntiles; ++j) {
      const int st = j % B3_NST;
      mbar_wait(&kv_empty[st], ((j / B3_NST) & 1) ^ 1);
      const int k0 = s0 + j * B_K;
      uint8_t* kd = sm + st * L::STAGE;
      mbar_arrive_expect_tx(&kv_full[st], L::STAGE);
      for (int sub = 0; sub < NSUB; ++sub) {
        tma_load_2d(kd + sub * SUB64, &tm_k, &kv_full[st], kvh * HD + 64 * sub, k0);
        tma_load_2d(kd + NSUB * SUB64 + sub * SUB64, &tm_v, &kv_full[st], kvh * HD + 64 * sub,
                    k0);
      }
    }
  } else if (warp == 1) {  // MMA: whole warp, uniform descriptors, elected issue
    constexpr uint32_t idesc_s = umma_idesc_bf16(B_Q, B_K, 0, 0);
    constexpr uint32_t idesc_q = umma_idesc_bf16(B_Q, HD, 0, 1);
    auto issue_sdp = [&](int j) {
      const int b = j & 1;
      mbar_wait(&kv_full[j % B3_NST], (j / B3_NST) & 1);
      tc_fence_after();
      const uint32_t k_addr = smem_u32(sm + (j % B3_NST) * L::STAGE);
      const uint32_t v_addr = k_addr + NSUB * SUB64;
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t okv = (kk >> 2) * SUB64 + (kk & 3) * 32;
          umma_f16_ts(tmem + TS + b * 128, tmem + TQ + kk * 8,
                      umma_desc_sw128(k_addr + okv, 16, 1024), idesc_s, kk != 0);
          umma_f16_ts(tmem + TS + b * 128 + 64, tmem + TDO + kk * 8,
                      umma_desc_sw128(v_addr + okv, 16, 1024), idesc_s, kk != 0);
        }
        umma_commit(&sd_full[b]);
      }
      __syncwarp();
    };
    auto issue_dq = [&](int j) {
      const int b = j & 1;
      mbar_wait(&ds_full[b], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t k_addr = smem_u32(sm + (j % B3_NST) * L::STAGE);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < B_K / 16; ++kk) {  // dS keys 16kk..: cols 0,8 | 32,40
          const uint32_t a = tmem + TS + b * 128 + (kk < 2 ? kk * 8 : 32 + (kk - 2) * 8);
          umma_f16_ts(tmem + TDQ, a, umma_desc_sw128(k_addr + kk * 2048, SUB64, 1024), idesc_q,
                      (j | kk) != 0);
        }
        umma_commit(&kv_empty[j % B3_NST]);
      }
      __syncwarp();
    };
    mbar_wait(q_ready, 0);
    tc_fence_after();
    issue_sdp(0);
    for (int j = 0; j < ntiles; ++j) {
      if (j + 1 < ntiles) issue_sdp(j + 1);  // S/dP[b^1] free: dQ(j-1) issued before it
      issue_dq(j);
    }
    if (elect_one()) umma_commit(dq_done);
    __syncwarp();
  } else if (warp >= 4) {
    // 8 softmax warps: lane quarter = warp % 4 (query rows), half = 32-key half
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int r = quarter * 32 + lane;
    const int qrow = q0 + r;
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    // stage Q (half 0) or dO (half 1) row r into TMEM as bf16 pairs
    {
      const bf16* src = half == 0 ? q + (long long)qrow * ldq + (long long)h * HD
                                  : dout + (long long)qrow * lddo + (long long)h * HD;
      const uint32_t col = half == 0 ? TQ : TDO;
#pragma unroll
      for (int c = 0; c < HD / 2; c += 16) {  // 16 columns = 32 bf16 = 4 x 16 B
        uint32_t v[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 u = *reinterpret_cast<const uint4*>(src + 2 * c + 8 * i);
          v[4 * i] = u.x;
          v[4 * i + 1] = u.y;
          v[4 * i + 2] = u.z;
          v[4 * i + 3] = u.w;
        }
        tmem_st_32x32b_x16(lane_base + col + c, v);
      }
      tmem_st_wait_all();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_ready);
    }
    const float sl2 = scale * kLog2e;
    const float lse2 = lse[(long long)h * T + qrow] * kLog2e;
    const float dl = delta[(long long)h * T + qrow];
    for (int j = 0; j < ntiles; ++j) {
      const int b = j & 1;
      mbar_wait(&sd_full[b], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[32], dpv[32], pk[16];
      tmem_ld_32x32b_x32(lane_base + TS + b * 128 + half * 32, sv);
      tmem_ld_32x32b_x32(lane_base + TS + b * 128 + 64 + half * 32, dpv);
      tmem_ld_wait();
      const int kbase = s0 + j * B_K + half * 32;  // first key of these columns
      const bool diag = kbase + 31 > q0;
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float p0 = ex2b(fmaf(__uint_as_float(sv[i]), sl2, -lse2));
        float p1 = ex2b(fmaf(__uint_as_float(sv[i + 1]), sl2, -lse2));
        if (diag) {
          if (kbase + i > qrow) p0 = 0.f;
          if (kbase + i + 1 > qrow) p1 = 0.f;
        }
        pk[i / 2] = pack_bf16x2(p0 * (__uint_as_float(dpv[i]) - dl),
                                p1 * (__uint_as_float(dpv[i + 1]) - dl));
      }
      tmem_st_32x32b_x16(lane_base + TS + b * 128 + half * 32, pk);  // over own read columns
      tmem_st_wait_all();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ds_full[b]);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    bf16* dqr = dq + (long long)qrow * lddq + (long long)h * HD;
#pragma unroll 1
    for (int c = half * (HD / 2); c < (half + 1) * (HD / 2); c += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(lane_base + TDQ + c, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 u;
        u.x = pack_bf16x2(__uint_as_float(v[i]) * scale, __uint_as_float(v[i + 1]) * scale);
        u.y = pack_bf16x2(__uint_as_float(v[i + 2]) * scale, __uint_as_float(v[i + 3]) * scale);
        u.z = pack_bf16x2(__uint_as_float(v[i + 4]) * scale, __uint_as_float(v[i + 5]) * scale);
        u.w = pack_bf16x2(__uint_as_float(v[i + 6]) * scale, __uint_as_float(v[i + 7]) * scale);
        *reinterpret_cast<uint4*>(dqr + c + i) = u;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// delta[h, t] = sum_d dO[t,h,d] * O[t,h,d]; one warp per (t, h), 16-byte loads
// (and, when nlse2 is given, nlse2[h, t] = -lse[h, t] * log2(e) for the fused kernel)
template <int HD>
__global__ void delta_kernel(const bf16* __restrict__ o, long long ldo, const bf16* __restrict__ d,
                             long long lddo, float* __restrict__ delta, int T, int nq,
                             const float* __restrict__ lse, float* __restrict__ nlse2) {
  const long long w = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (w >= (long long)T * nq) return;
  const int t = (int)(w / nq), h = (int)(w % nq);
  float acc = 0.f;
  for (int c = lane * 8; c < HD; c += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(o + (long long)t * ldo + h * HD + c);
    const uint4 b = *reinterpret_cast<const uint4*>(d + (long long)t * lddo + h * HD + c);
    const bf16* pa = reinterpret_cast<const bf16*>(&a);
    const bf16* pb = reinterpret_cast<const bf16*>(&b);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += __bfloat162float(pa[i]) * __bfloat162float(pb[i]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    delta[(long long)h * T + t] = acc;
    if (nlse2) nlse2[(long long)h * T + t] = -lse[(long long)h * T + t] * kLog2e;
  }
}

// dk/dv (bf16, strided) = dk_acc/dv_acc (fp32 [T, nk*HD])
__global__ void dkv_cast_kernel(const float* __restrict__ dka, const float* __restrict__ dva,
                                bf16* __restrict__ dk, long long lddk, bf16* __restrict__ dv,
                                long long lddv, int T, int cols) {
  const long long n4 = (long long)T * cols / 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i * 4, t = e / cols;
    const int c = (int)(e % cols);
    const float4 a = reinterpret_cast<const float4*>(dka)[i];
    const float4 b = reinterpret_cast<const float4*>(dva)[i];
    uint2 ua, ub;
    ua.x = pack_bf16x2(a.x, a.y);
    ua.y = pack_bf16x2(a.z, a.w);
    ub.x = pack_bf16x2(b.x, b.y);
    ub.y = pack_bf16x2(b.z, b.w);
    *reinterpret_cast<uint2*>(dk + t * lddk + c) = ua;
    *reinterpret_cast<uint2*>(dv + t * lddv + c) = ub;
  }
}

// dq[t, c] (bf16, strided) = scale * acc[c, t]: transpose of the d-major fp32
// accumulator through a 32 x 33 shared tile (block 32 x 8)
__global__ void dq_cast_kernel(const float* __restrict__ acc, bf16* __restrict__ dq, long long lddq,
                               int T, int cols, float scale) {
  __shared__ float tile[32][33];
  const int t0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int i = 0; i < 32; i += 8) tile[ty + i][tx] = acc[(long long)(c0 + ty + i) * T + t0 + tx];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 32; i += 8)
    dq[(long long)(t0 + ty + i) * lddq + c0 + tx] = __float2bfloat16_rn(tile[tx][ty + i] * scale);
}

// ---- host ------------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    return reinterpret_cast<EncodeFn>(ptr);
  }();
  return fn;
}
bool map2d(CUtensorMap* m, const void* base, long long rows, long long cols, long long ld,
           int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  EncodeFn fn = encode_fn();
  return fn && fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                   CUDA_SUCCESS;
}

bool map_f32(CUtensorMap* m, const void* base, long long rows, long long cols, long long ld) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  EncodeFn fn = encode_fn();
  return fn && fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                   CUDA_SUCCESS;
}

template <class K>
bool set_smem(K kern, int bytes) {
  return ensure_smem_t(kern, bytes);
}

template <int HD>
int bwd_tc(const void* q, long long ldq, const void* k, long long ldk, const void* v,
           long long ldv, const void* o, long long ldo, const void* dout, long long lddo,
           const float* lse, void* dq, long long lddq, void* dk, long long lddk, void* dv,
           long long lddv, float* delta, float* dkv_acc, int T, int seq, int nq, int nk,
           float scale, cudaStream_t s) {
  const long long warps = (long long)T * nq;
  const int G = nq / nk;
  const bool fused = HD == 128 && G % 2 == 0;
  // fused path workspace: fp32 d-major dQ^T accumulator [nq*HD, T], then
  // -lse*log2(e) [nq, T]
  const long long qn = (long long)T * nq * HD;
  float* dq_acc = nullptr;
  if (fused) {
    Workspace* w = stream_workspace(s, WS_ATTN_DQ, sizeof(float) * (size_t)(qn + warps));
    if (!w) return RP_E_CUDA;
    dq_acc = static_cast<float*>(w->p);
  }
  float* nlse2 = fused ? dq_acc + qn : nullptr;
  delta_kernel<HD><<<(int)((warps + 7) / 8), 256, 0, s>>>((const bf16*)o, ldo, (const bf16*)dout,
                                                         lddo, delta, T, nq, lse, nlse2);
  CUtensorMap mk128, mv128, mq64, mdo64;
  if (!map2d(&mk128, k, T, (long long)nk * HD, ldk, 128) ||
      !map2d(&mv128, v, T, (long long)nk * HD, ldv, 128) ||
      !map2d(&mq64, q, T, (long long)nq * HD, ldq, 64) ||
      !map2d(&mdo64, dout, T, (long long)nq * HD, lddo, 64))
    return RP_E_CUDA;
  const long long acc_n = (long long)T * nk * HD;
  if (fused) {  // dK/dV/dQ in one kernel (A4)
    CUtensorMap mdq;
    if (!map_f32(&mdq, dq_acc, (long long)nq * HD, T, T))  // d-major [nq*HD, T]
      return RP_E_CUDA;
    if (cudaMemsetAsync(dq_acc, 0, sizeof(float) * qn, s) != cudaSuccess) return RP_E_CUDA;
    // GQA partials of dK/dV: G = 2 both heads share the CTA (bf16 straight
    // from TMEM); G = 4 a 2-CTA cluster sums over DSMEM; G >= 8 fp32 atomics
    const int cl = G == 2 ? 1 : G == 4 ? 2 : 0;
    auto go = [&](auto kern, int cluster) -> cudaError_t {
      if (!set_smem(kern, Dkv4Smem<HD>::BYTES)) return cudaErrorInvalidValue;
      cudaLaunchConfig_t c = {};
      c.gridDim = dim3(nq / 2, T / A_BK, 1);
      c.blockDim = dim3(A4_THREADS, 1, 1);
      c.dynamicSmemBytes = Dkv4Smem<HD>::BYTES;
      c.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      c.attrs = at;
      c.numAttrs = 1;
      return cudaLaunchKernelEx(&c, kern, mk128, mv128, mq64, mdo64, mdq, (const float*)nlse2,
                                (const float*)delta,
                                dkv_acc, dkv_acc + acc_n, (bf16*)dk, (long long)lddk, (bf16*)dv,
                                (long long)lddv, T, seq, nq, nk, scale);
    };
    if (cl == 0 &&
        cudaMemsetAsync(dkv_acc, 0, sizeof(float) * 2 * acc_n, s) != cudaSuccess)
      return RP_E_CUDA;
    cudaError_t e = cl == 2   ? go(attn_bwd_fused_kernel<HD, 2>, 2)
                    : cl == 1 ? go(attn_bwd_fused_kernel<HD, 1>, 1)
                              : go(attn_bwd_fused_kernel<HD, 0>, 1);
    if (e != cudaSuccess) return RP_E_CUDA;
    if (cl == 0)
      dkv_cast_kernel<<<148 * 8, 256, 0, s>>>(dkv_acc, dkv_acc + acc_n, (bf16*)dk, lddk, (bf16*)dv,
                                              lddv, T, nk * HD);
    dq_cast_kernel<<<dim3(T / 32, nq * HD / 32), dim3(32, 8), 0, s>>>(dq_acc, (bf16*)dq, lddq, T,
                                                                      nq * HD, scale);
    return cudaGetLastError() == cudaSuccess ? RP_OK : RP_E_CUDA;
  }
  // two-kernel path: dK/dV (A2 for even groups, A otherwise) + dQ (B3)
  if (cudaMemsetAsync(dkv_acc, 0, sizeof(float) * 2 * acc_n, s) != cudaSuccess) return RP_E_CUDA;
  if (G % 2 == 0) {
    if (!set_smem(attn_bwd_dkv_pp_kernel<HD>, Dkv2Smem<HD>::BYTES)) return RP_E_CUDA;
    attn_bwd_dkv_pp_kernel<HD><<<dim3(nq / 2, T / A_BK), A2_THREADS, Dkv2Smem<HD>::BYTES, s>>>(
        mk128, mv128, mq64, mdo64, lse, delta, dkv_acc, dkv_acc + acc_n, T, seq, nq, nk, scale);
  } else {
    if (!set_smem(attn_bwd_dkv_kernel<HD>, DkvSmem<HD>::BYTES)) return RP_E_CUDA;
    attn_bwd_dkv_kernel<HD><<<dim3(nq, T / A_BK), 384, DkvSmem<HD>::BYTES, s>>>(
        mk128, mv128, mq64, mdo64, lse, delta, dkv_acc, dkv_acc + acc_n, T, seq, nq, nk, scale);
  }
  dkv_cast_kernel<<<148 * 8, 256, 0, s>>>(dkv_acc, dkv_acc + acc_n, (bf16*)dk, lddk, (bf16*)dv,
                                          lddv, T, nk * HD);
  CUtensorMap mk64, mv64;
  if (!map2d(&mk64, k, T, (long long)nk * HD, ldk, 64) ||
      !map2d(&mv64, v, T, (long long)nk * HD, ldv, 64))
    return RP_E_CUDA;
  if (!set_smem(attn_bwd_dq3_kernel<HD>, Dq3Smem<HD>::BYTES)) return RP_E_CUDA;
  attn_bwd_dq3_kernel<HD><<<dim3(nq, T / B_Q), 384, Dq3Smem<HD>::BYTES, s>>>(
      (const bf16*)q, ldq, (const bf16*)dout, lddo, mk64, mv64, lse, delta, (bf16*)dq, lddq, T,
      seq, nq, nk, scale);
  return cudaGetLastError() == cudaSuccess ? RP_OK : RP_E_CUDA;
}

}  // namespace
}  // namespace rp

// tcgen05 backward: dq/dk/dv (bf16) from q/k/v/o/dO/lse; `delta` is an fp32
// [nq, T] workspace, dkv_acc an fp32 [2, T, nk*head_dim] one. dK/dV (and, on
// the default fused path, dQ) are reduced in fp32 through L2 atomics / TMA
// reduce-adds, so bits can vary run to run. Layouts as rp_attn_fwd_tc.
extern "C" __attribute__((visibility("default"))) int rp_attn_bwd_tc(
    const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
    const void* o, int64_t ldo, const void* dout, int64_t lddo, const float* lse, void* dq,
    int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv, float* delta, float* dkv_acc,
    int32_t T, int32_t seq, int32_t nq, int32_t nk, int32_t head_dim, float scale, void* stream) {
  if (T <= 0 || seq % 128 || T % seq || nk <= 0 || nq % nk || (head_dim != 64 && head_dim != 128))
    return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  return head_dim == 128
             ? rp::bwd_tc<128>(q, ldq, k, ldk, v, ldv, o, ldo, dout, lddo, lse, dq, lddq, dk, lddk,
                               dv, lddv, delta, dkv_acc, T, seq, nq, nk, scale, s)
             : rp::bwd_tc<64>(q, ldq, k, ldk, v, ldv, o, ldo, dout, lddo, lse, dq, lddq, dk, lddk,
                              dv, lddv, delta, dkv_acc, T, seq, nq, nk, scale, s);
}
