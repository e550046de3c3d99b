// Causal GQA flash attention FORWARD on the 5th-gen tensor cores (sm_100a).
//
// One CTA = 128 query rows x 1 head. Warp roles (192 threads):
//   w0  TMA producer: Q once, then K_j / V_j tiles (128 keys) into a 2-stage ring
//   w1  MMA issuer (one thread): S_j = Q K_j^T  (tcgen05.mma M128 N128, K=hd)
//       into a double-buffered TMEM S, then O += P_{j-1} V_{j-1} (M128 N=hd,
//       K=128 keys; P from shared memory, V as an MN-major operand) into TMEM O
//   w2-5 softmax: one thread per query row (TMEM lane), tcgen05.ld of the S row,
//       causal mask on the diagonal tile, exp2 with a lazily-updated running
//       max (O in TMEM is rescaled only when the max grows by > 2^8), P (bf16)
//       written to swizzled smem for the PV MMA; final O / l, bf16 store, LSE.
// S_{j+1} is issued before PV_j, so the tensor core computes the next scores
// while the softmax warps work on the current tile.
#include <cstdlib>

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

constexpr int TILE = 128;          // queries per CTA, keys per K/V tile
constexpr int SUB = TILE * 128;    // one 128-row x 64-col bf16 swizzled sub-tile (16 KB)

template <int HD>
struct FwdSmem {
  static constexpr int NSUB = HD / 64;
  static constexpr int Q = 0;
  static constexpr int K0 = Q + NSUB * SUB;
  static constexpr int V0 = K0 + NSUB * SUB;
  static constexpr int K1 = V0 + NSUB * SUB;
  static constexpr int V1 = K1 + NSUB * SUB;
  static constexpr int P = V1 + NSUB * SUB;
  static constexpr int BAR = P + 2 * SUB;
  static constexpr int BYTES = BAR + 256 + 1024;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

template <int HD>
__global__ void __launch_bounds__(192, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, bf16* __restrict__ o,
                       long long ldo, float* __restrict__ lse, int T, int seq, int nq, int nk,
                       float scale) {
  using L = FwdSmem<HD>;
  constexpr int NSUB = L::NSUB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;     // [2]
  uint64_t* v_full = bar + 3;     // [2]
  uint64_t* kv_empty = bar + 5;   // [2]
  uint64_t* s_full = bar + 7;     // [2]
  uint64_t* s_free = bar + 9;     // [2]
  uint64_t* p_full = bar + 11;
  uint64_t* o_done = bar + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 13);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qblocks = T / TILE;
  const int qb = causal_block(blockIdx.y, qblocks, seq / TILE, true);  // heaviest first
  const int h = blockIdx.x, kvh = h / (nq / nk);
  const int q0 = qb * TILE;
  const int s0 = (q0 / seq) * seq;
  const int ntiles = (q0 - s0) / TILE + 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t TM_O = 256;

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ TMA producer
    mbar_arrive_expect_tx(q_full, NSUB * SUB);
    for (int sub = 0; sub < NSUB; ++sub)
      tma_load_2d(sm + L::Q + sub * SUB, &tm_q, q_full, h * HD + 64 * sub, q0);
    for (int j = 0; j < ntiles; ++j) {
      const int st = j & 1;
      mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
      const int k0 = s0 + j * TILE;
      uint8_t* kd = sm + (st ? L::K1 : L::K0);
      uint8_t* vd = sm + (st ? L::V1 : L::V0);
      mbar_arrive_expect_tx(&k_full[st], NSUB * SUB);
      for (int sub = 0; sub < NSUB; ++sub)
        tma_load_2d(kd + sub * SUB, &tm_k, &k_full[st], kvh * HD + 64 * sub, k0);
      mbar_arrive_expect_tx(&v_full[st], NSUB * SUB);
      for (int sub = 0; sub < NSUB; ++sub)
        tma_load_2d(vd + sub * SUB, &tm_v, &v_full[st], kvh * HD + 64 * sub, k0);
    }
  } else if (warp == 1 && lane == 0) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = umma_idesc_bf16(TILE, TILE, 0, 0);
    constexpr uint32_t idesc_o = umma_idesc_bf16(TILE, HD, 0, 1);
    const uint32_t q_addr = smem_u32(sm + L::Q);
    const uint32_t p_addr = smem_u32(sm + L::P);
    auto issue_pv = [&](int j) {
      const int st = j & 1;
      mbar_wait(p_full, j & 1);
      mbar_wait(&v_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t v_addr = smem_u32(sm + (st ? L::V1 : L::V0));
#pragma unroll
      for (int kk = 0; kk < TILE / 16; ++kk) {
        const uint64_t ad = umma_desc_sw128(p_addr + (kk >> 2) * SUB + (kk & 3) * 32, 16, 1024);
        const uint64_t bd = umma_desc_sw128(v_addr + kk * 2048, SUB, 1024);
        umma_f16(tmem + TM_O, ad, bd, idesc_o, (j | kk) != 0);
      }
      umma_commit(o_done);
      umma_commit(&kv_empty[st]);
    };
    mbar_wait(q_full, 0);
    for (int j = 0; j < ntiles; ++j) {
      const int st = j & 1;
      mbar_wait(&k_full[st], (j >> 1) & 1);
      if (j >= 2) mbar_wait(&s_free[st], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t k_addr = smem_u32(sm + (st ? L::K1 : L::K0));
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const uint64_t ad = umma_desc_sw128(q_addr + (kk >> 2) * SUB + (kk & 3) * 32, 16, 1024);
        const uint64_t bd = umma_desc_sw128(k_addr + (kk >> 2) * SUB + (kk & 3) * 32, 16, 1024);
        umma_f16(tmem + st * TILE, ad, bd, idesc_s, kk != 0);
      }
      umma_commit(&s_full[st]);
      if (j >= 1) issue_pv(j - 1);
    }
    issue_pv(ntiles - 1);
  } else if (warp >= 2) {
    // ------------------------------------------------------------ softmax
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // query row within the tile
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    const float sl2 = scale * 1.4426950408889634f;
    float m = 0.f, l = 0.f;
    uint8_t* p_row = sm + L::P + (r >> 3) * 1024 + (r & 7) * 128;
    for (int j = 0; j < ntiles; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[TILE];
#pragma unroll
      for (int c = 0; c < TILE; c += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(lane_base + st * TILE + c, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(v[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[st]);
      if (j == ntiles - 1) {  // diagonal tile: key c > query r is masked
#pragma unroll
        for (int c = 0; c < TILE; ++c)
          if (c > r) s[c] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < TILE; ++c) mx = fmaxf(mx, s[c]);
      const float mxs = mx * sl2;
      bool o_ready = false;
      if (j == 0) {
        m = mxs;
      } else if (__any_sync(0xffffffffu, mxs > m + 8.f)) {
        // some row's max grew by > 2^8: the whole warp rescales its O rows
        // (tcgen05.ld/st are warp-collective) after PV_{j-1}, and l
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
        o_ready = true;
        const float m_new = fmaxf(m, mxs);
        const float f = ex2(m - m_new);
        m = m_new;
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(lane_base + TM_O + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * f);
          tmem_st_32x32b_x32(lane_base + TM_O + c, v);
        }
        tmem_st_wait();
        l *= f;
      }
      float lsum = 0.f;
      uint32_t pk[TILE / 2];
#pragma unroll
      for (int c = 0; c < TILE; c += 2) {
        const float p0 = ex2(fmaf(s[c], sl2, -m));
        const float p1 = ex2(fmaf(s[c + 1], sl2, -m));
        lsum += p0 + p1;
        pk[c / 2] = pack_bf16x2(p0, p1);
      }
      l += lsum;
      if (j >= 1 && !o_ready) {  // PV_{j-1} must be done reading the P buffer
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
      }
#pragma unroll
      for (int ch = 0; ch < TILE / 8; ++ch) {  // 16-byte chunks of the swizzled row
        const int sub = ch >> 3, c8 = ch & 7;
        uint4 u = make_uint4(pk[ch * 4], pk[ch * 4 + 1], pk[ch * 4 + 2], pk[ch * 4 + 3]);
        *reinterpret_cast<uint4*>(p_row + sub * SUB + ((c8 ^ (r & 7)) << 4)) = u;
      }
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16, LSE
    mbar_wait(o_done, (ntiles - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const int qrow = q0 + r;
    bf16* orow = o + (long long)qrow * ldo + (long long)h * HD;
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(lane_base + TM_O + c, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 u;
        u.x = pack_bf16x2(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv);
        u.y = pack_bf16x2(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv);
        u.z = pack_bf16x2(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv);
        u.w = pack_bf16x2(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv);
        *reinterpret_cast<uint4*>(orow + c + i) = u;
      }
    }
    lse[(long long)h * T + qrow] = (m + __log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ======================================================================
// Ping-pong variant: one CTA = 128 query rows x TWO query heads of the same
// KV group (GQA), so both Q tiles consume the same K/V tiles (loaded once)
// and two softmax warpgroups alternate with the tensor core:
//   w0      TMA: Q0, Q1 once; then K_0, V_0, K_1, V_1, ... through a 4-slot ring
//   w1      MMA: S0_{j+1} = Q0 K^T and S1_{j+1} = Q1 K^T interleaved with
//           O0 += P0_j V_j and O1 += P1_j V_j (TMEM: S0 | S1 | O0 | O1)
//   w4-7    softmax of head 0 (thread = query row),  w8-11  softmax of head 1
// While one warpgroup turns its S into P the tensor core runs the other
// head's MMAs. P goes back into the TMEM columns of its S (bf16 pairs) and
// feeds the PV MMA as a TMEM A operand (no P traffic through shared memory,
// whose port the N=128 SS MMAs already saturate).
//
// The chain of one head is softmax_j -> PV_j -> S_{j+1} -> softmax_{j+1}, so
// the tensor core idles unless a softmax pass finishes within the other
// head's PV + S (1024 MMA cycles). At 16 ex2/clk/SM the MUFU alone needs
// 1024 cycles for a 128x128 tile, so the pass is shortened three ways:
//   * a quarter of the exponentials run on the FMA pipe (ex2_fma2: rint by
//     the 1.5*2^23 add, degree-3 polynomial, 2^n added into the exponent;
//     rel. error 7.5e-5, far below the bf16 rounding of P; measured 0.1195 ms
//     vs 0.1208 all-MUFU and 0.1218 with half emulated,
//     profiles/r02_attn_fwd_variants.jsonl);
//   * P is published in two halves: PV's first four K=16 steps run while the
//     warpgroup computes the second half;
//   * the row max uses 3-input FMNMX3; the four S loads share one wait.
// Registers: the producer/MMA warpgroup gives its registers to the softmax
// warpgroups (setmaxnreg 56 / 224), so the 128-float row never spills.
constexpr int PP_THREADS = 384;

template <int HD>
struct PpSmem {
  static constexpr int NSUB = HD / 64;
  static constexpr int QT = NSUB * SUB;       // one Q tile (128 rows x HD)
  static constexpr int KVT = NSUB * SUB;      // one K or V tile (128 keys x HD)
  static constexpr int NSLOT = 4;             // K/V ring slots
  static constexpr int Q0 = 0;
  static constexpr int RING = Q0 + 2 * QT;
  static constexpr int BAR = RING + NSLOT * KVT;
  static constexpr int BYTES = BAR + 256 + 1024;
  static_assert(BYTES <= 232448, "exceeds 227 KB of shared memory");
};

// 2^x for -125 <= x (clamped) and x < 2^22, on the FMA/ALU pipes.
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 rnd = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = __fadd2_rn(x, rnd);                      // mantissa low bits = rint(x)
  const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-n.x, -n.y));  // [-0.5, 0.5]
  float2 p = __ffma2_rn(f, make_float2(0.05517167f, 0.05517167f),
                        make_float2(0.24261113f, 0.24261113f));
  p = __ffma2_rn(p, f, make_float2(0.69326097f, 0.69326097f));
  p = __ffma2_rn(p, f, make_float2(0.99992806f, 0.99992806f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// EMU: pairs out of every four (8 probabilities) computed by ex2_fma2.
template <int HD, int EMU>
__global__ void __launch_bounds__(PP_THREADS, 1)
    attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, bf16* __restrict__ o,
                       long long ldo, float* __restrict__ lse, int T, int seq, int nq, int nk,
                       float scale) {
  using L = PpSmem<HD>;
  constexpr int NS = L::NSLOT;
  constexpr int NSUB = L::NSUB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;        // [NS]
  uint64_t* kv_empty = bar + 1 + NS;  // [NS]
  uint64_t* s_full = kv_empty + NS;   // [2] per head
  uint64_t* p_half = s_full + 2;      // [2 heads][2 halves]
  uint64_t* o_done = p_half + 4;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int qblocks = T / TILE;
  const int qb = causal_block(blockIdx.y, qblocks, seq / TILE, true);  // heaviest first
  const int h0 = 2 * (int)blockIdx.x;  // heads h0, h0+1 share a KV head
  const int kvh = h0 / (nq / nk);
  const int q0 = qb * TILE;
  const int s0 = (q0 / seq) * seq;
  const int ntiles = (q0 - s0) / TILE + 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&o_done[i], 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&p_half[i], 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S_w at w*128, O_w at 256 + w*HD

  if (warp < 4) {
    setmaxnreg_dec<56>();
    if (warp == 0 && lane == 0) {
      // ---------------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(q_full, 2 * L::QT);
      for (int w = 0; w < 2; ++w)
        for (int sub = 0; sub < NSUB; ++sub)
          tma_load_2d(sm + L::Q0 + w * L::QT + sub * SUB, &tm_q, q_full,
                      (h0 + w) * HD + 64 * sub, q0);
      for (int idx = 0; idx < 2 * ntiles; ++idx) {
        const int slot = idx % NS;
        mbar_wait(&kv_empty[slot], ((idx / NS) & 1) ^ 1);
        const int k0 = s0 + (idx >> 1) * TILE;
        uint8_t* dst = sm + L::RING + slot * L::KVT;
        mbar_arrive_expect_tx(&kv_full[slot], L::KVT);
        const CUtensorMap* map = (idx & 1) ? &tm_v : &tm_k;
        for (int sub = 0; sub < NSUB; ++sub)
          tma_load_2d(dst + sub * SUB, map, &kv_full[slot], kvh * HD + 64 * sub, k0);
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      // (whole warp: uniform descriptors; one elected lane issues)
      constexpr uint32_t idesc_s = umma_idesc_bf16(TILE, TILE, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(TILE, HD, 0, 1);
      const uint32_t q_addr = smem_u32(sm + L::Q0);
      auto ring = [&](int idx) { return smem_u32(sm + L::RING + (idx % NS) * L::KVT); };
      auto wait_kv = [&](int idx) { mbar_wait(&kv_full[idx % NS], (idx / NS) & 1); };
      auto issue_s = [&](int w, int j) {  // S_w = Q_w K_j^T
        const uint32_t qa = q_addr + w * L::QT, ka = ring(2 * j);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * SUB + (kk & 3) * 32;
            umma_f16(tmem + w * TILE, umma_desc_sw128(qa + off, 16, 1024),
                     umma_desc_sw128(ka + off, 16, 1024), idesc_s, kk != 0);
          }
          umma_commit(&s_full[w]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int w, int j) {  // O_w += P_w V_j, one half of the keys at a time
        const uint32_t va = ring(2 * j + 1);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          mbar_wait(&p_half[2 * w + half], j & 1);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = half * 4; kk < half * 4 + 4; ++kk)  // P: 8 bf16-pair columns per K=16
              umma_f16_ts(tmem + 256 + w * HD, tmem + w * TILE + kk * 8,
                          umma_desc_sw128(va + kk * 2048, SUB, 1024), idesc_o, (j | kk) != 0);
            if (half) umma_commit(&o_done[w]);
          }
          __syncwarp();
        }
      };
      mbar_wait(q_full, 0);
      wait_kv(0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      if (elect_one()) umma_commit(&kv_empty[0]);
      __syncwarp();
      for (int j = 0; j < ntiles; ++j) {
        wait_kv(2 * j + 1);
        tc_fence_after();
        issue_pv(0, j);
        const bool more = j + 1 < ntiles;
        if (more) {
          wait_kv(2 * j + 2);
          tc_fence_after();
          issue_s(0, j + 1);  // S0 was read before P0_j was published
        }
        issue_pv(1, j);
        if (elect_one()) umma_commit(&kv_empty[(2 * j + 1) % NS]);
        __syncwarp();
        if (more) {
          issue_s(1, j + 1);
          if (elect_one()) umma_commit(&kv_empty[(2 * j + 2) % NS]);
          __syncwarp();
        }
      }
    }
  } else {
    setmaxnreg_inc<224>();
    // ------------------------------------------------------------ softmax
    const int w = (warp - 4) >> 2;      // head slot of this warpgroup
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // query row within the tile
    const uint32_t lane_base = tmem + (uint32_t(quarter * 32) << 16);
    const uint32_t s_col = w * TILE, o_col = 256 + w * HD;
    const float sl2 = scale * 1.4426950408889634f;
    float m = 0.f, l = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const bool diag = j == ntiles - 1;
      mbar_wait(&s_full[w], j & 1);
      tc_fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(lane_base + s_col + 32 * c, sr[c]);
      tmem_ld_wait();
      float s[TILE];
#pragma unroll
      for (int c = 0; c < TILE; ++c) s[c] = __uint_as_float(sr[c >> 5][c & 31]);
      if (diag) {  // diagonal tile: key c > query r is masked
#pragma unroll
        for (int c = 0; c < TILE; ++c)
          if (c > r) s[c] = -INFINITY;
      }
      float mx8[8];  // 8 independent max chains of 3-input max
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        mx8[i] = s[i];
#pragma unroll
        for (int k = 0; k < 7; ++k) mx8[i] = fmax3(mx8[i], s[8 + 16 * k + i], s[16 + 16 * k + i]);
        mx8[i] = fmaxf(mx8[i], s[120 + i]);
      }
      const float mx = fmaxf(fmax3(mx8[0], mx8[1], mx8[2]),
                             fmaxf(fmax3(mx8[3], mx8[4], mx8[5]), fmax3(mx8[6], mx8[7], mx8[7])));
      const float mxs = mx * sl2;
      if (j == 0) {
        m = mxs;
      } else if (__any_sync(0xffffffffu, mxs > m + 8.f)) {
        // some row's max grew by > 2^8: rescale this warp's O rows after PV_{j-1}
        mbar_wait(&o_done[w], (j - 1) & 1);
        tc_fence_after();
        const float m_new = fmaxf(m, mxs);
        const float f = ex2(m - m_new);
        m = m_new;
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(lane_base + o_col + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * f);
          tmem_st_32x32b_x32(lane_base + o_col + c, v);
        }
        tmem_st_wait();
        l *= f;
      }
      // (PV_{j-1} read P_{j-1} from these TMEM columns before S_j overwrote them)
      // P = 2^(s*scale*log2e - m); four independent row-sum chains
      float2 lsum4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
      const float2 sl2v = make_float2(sl2, sl2), negm = make_float2(-m, -m);
      auto exp_pass = [&]<bool E>() {
        uint32_t pt[16];  // 32 probabilities = 16 TMEM columns per store
#pragma unroll
        for (int ch = 0; ch < TILE / 8; ++ch) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x =
                __ffma2_rn(make_float2(s[ch * 8 + 2 * e], s[ch * 8 + 2 * e + 1]), sl2v, negm);
            const float2 pv = (E && e >= 4 - EMU) ? ex2_fma2(x) : make_float2(ex2(x.x), ex2(x.y));
            lsum4[e] = __fadd2_rn(lsum4[e], pv);
            pt[(ch & 3) * 4 + e] = pack_bf16x2(pv.x, pv.y);
          }
          if ((ch & 3) == 3) tmem_st_32x32b_x16(lane_base + s_col + (ch >> 2) * 16, pt);
          if ((ch & 7) == 7) {  // one half of P (64 keys) is in TMEM: release it to PV
            tmem_st_wait_all();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_half[2 * w + (ch >> 3)]);
          }
        }
      };
      if (diag) exp_pass.template operator()<false>();
      else exp_pass.template operator()<true>();
      const float2 ls = __fadd2_rn(__fadd2_rn(lsum4[0], lsum4[1]), __fadd2_rn(lsum4[2], lsum4[3]));
      l += ls.x + ls.y;
    }
    // epilogue: O / l -> bf16, LSE
    mbar_wait(&o_done[w], (ntiles - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const int qrow = q0 + r;
    const int h = h0 + w;
    bf16* orow = o + (long long)qrow * ldo + (long long)h * HD;
#pragma unroll 1
    for (int c = 0; c < HD; c += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(lane_base + o_col + c, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 u;
        u.x = pack_bf16x2(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv);
        u.y = pack_bf16x2(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv);
        u.z = pack_bf16x2(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv);
        u.w = pack_bf16x2(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv);
        *reinterpret_cast<uint4*>(orow + c + i) = u;
      }
    }
    lse[(long long)h * T + qrow] = (m + __log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---- host ----------------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode() {
  static EncodeFn fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    return reinterpret_cast<EncodeFn>(ptr);
  }();
  return fn;
}
// [rows, cols] bf16 (row pitch ld elements), box {64 cols, 128 rows}, SW128
bool map_tile(CUtensorMap* m, const void* base, long long rows, long long cols, long long ld) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  return encode() &&
         encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD>
int fwd_tc(const void* q, long long ldq, const void* k, long long ldk, const void* v,
           long long ldv, void* o, long long ldo, float* lse, int T, int seq, int nq, int nk,
           float scale, cudaStream_t s) {
  CUtensorMap mq, mk, mv;
  if (!map_tile(&mq, q, T, (long long)nq * HD, ldq) || !map_tile(&mk, k, T, (long long)nk * HD, ldk) ||
      !map_tile(&mv, v, T, (long long)nk * HD, ldv))
    return RP_E_CUDA;
  if ((nq / nk) % 2 == 0) {  // two heads of one KV group per CTA
    auto kern = attn_fwd_pp_kernel<HD, 1>;
    const int bytes = PpSmem<HD>::BYTES;
    if (!ensure_smem_t(kern, bytes)) return RP_E_CUDA;
    dim3 grid(nq / 2, T / TILE);
    kern<<<grid, PP_THREADS, bytes, s>>>(mq, mk, mv, (bf16*)o, ldo, lse, T, seq, nq, nk, scale);
    return cudaGetLastError() == cudaSuccess ? RP_OK : RP_E_CUDA;
  }
  auto kern = attn_fwd_tc_kernel<HD>;
  if (!ensure_smem_t(kern, FwdSmem<HD>::BYTES)) return RP_E_CUDA;
  dim3 grid(nq, T / TILE);
  kern<<<grid, 192, FwdSmem<HD>::BYTES, s>>>(mq, mk, mv, (bf16*)o, ldo, lse, T, seq, nq, nk, scale);
  return cudaGetLastError() == cudaSuccess ? RP_OK : RP_E_CUDA;
}

}  // namespace
}  // namespace rp

// tcgen05 forward (include/rp/kernels.h): 16-byte aligned q/k/v/o base
// pointers and pitches.
extern "C" __attribute__((visibility("default"))) int rp_attn_fwd_tc(
    const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv, void* o,
    int64_t ldo, float* lse, int32_t T, int32_t seq, int32_t nq, int32_t nk, int32_t head_dim,
    float scale, void* stream) {
  if (T <= 0 || seq % 128 || T % seq || nk <= 0 || nq % nk || (head_dim != 64 && head_dim != 128))
    return RP_E_INPUT;
  if ((ldq * 2) % 16 || (ldk * 2) % 16 || (ldv * 2) % 16 || (ldo * 2) % 16) return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  return head_dim == 128 ? rp::fwd_tc<128>(q, ldq, k, ldk, v, ldv, o, ldo, lse, T, seq, nq, nk, scale, s)
                         : rp::fwd_tc<64>(q, ldq, k, ldk, v, ldv, o, ldo, lse, T, seq, nq, nk, scale, s);
}
