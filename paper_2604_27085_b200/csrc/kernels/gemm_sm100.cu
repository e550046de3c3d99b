// Persistent warp-specialised bf16 GEMM for sm_100a (tcgen05 + TMEM + TMA).
//
//   D[M,N] (+)= A[M,K] . B[N,K]^T      bf16 inputs, fp32 accumulation in TMEM
//
// Each operand is K-major (row-major with K contiguous) or MN-major (K rows
// with M/N contiguous), so one kernel family covers the three GEMMs of every
// linear layer without materialised transposes:
//   forward  Y  = X  . W^T   A=X  K-major,  B=W  K-major
//   dgrad    dX = dY . W     A=dY K-major,  B=W  N-major
//   wgrad    dW += dY^T . X  A=dY M-major,  B=X  N-major   (fp32 accumulate)
//
// Tile 128x256x64, 4-stage TMA->smem ring (SWIZZLE_128B), one elected thread
// issues tcgen05.mma (M=128, N=256, K=16) into a double-buffered 2x256-column
// TMEM accumulator; 4 epilogue warps drain TMEM (tcgen05.ld 32x32b) while the
// next tile's MMAs run. Grid = min(tiles, #SMs), static round-robin tiles with
// M fastest so consecutive CTAs share the B panel in L2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels/launch_util.h"
#include "kernels/sm100.cuh"
#include "kernels/swiglu.cuh"
#include "rp/kernels.h"

namespace rp {
namespace {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_STAGE_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int NUM_THREADS = 256;             // w0 TMA, w1 MMA, w2 TMEM, w4-7 epilogue
constexpr int TMEM_COLS = 512;               // 2 x 256-column accumulators
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// EPI_SWIGLU_BWD: the accumulator is dact = dL/d(silu(g)*u) [M, N]; R holds
// gu = [g | u] ([M, 2N], pitch ldr) and D receives dgu = [dg | du] (pitch ldd)
// EPI_SWIGLU_FWD ("dual" gate/up GEMM, pair kernel only): B = W_gu [2N, K];
// the pair tile's two 128-row B halves are gate rows n0.. and up rows N+n0..,
// so each TMEM row holds g (cols 0-127) and u (cols 128-255) of the same
// outputs; the epilogue writes gu = [g | u] to D ([M, 2N]) and act =
// silu(g) * u to D2 ([M, N])
enum Epi : int { EPI_BF16 = 0, EPI_F32 = 1, EPI_F32_ACC = 2, EPI_SWIGLU_BWD = 3, EPI_SWIGLU_FWD = 4 };

struct Params {
  int M, N, K;
  void* D;
  long long ldd;
  const __nv_bfloat16* R;  // optional bf16 residual for EPI_BF16
  long long ldr;
  int vec;                 // 16-byte vector stores/loads legal for D (and R)
  int tma_out;             // fp32 D written through the TMA map (pair kernel)
  int tma_swiglu;          // EPI_SWIGLU_BWD through the EpiMaps (pair kernel)
  int trans;               // store D transposed: element (m, n) -> D[n * ldd + m] (skinny swap)
  // split-K of the last partial wave (pair kernel): work units [0, full) are
  // whole tiles, units beyond are the two K halves of tile full + (u-full)/2;
  // the first half parks its fp32 partial in `ws` and raises a per-warp flag
  // (= epoch), the second adds it in its epilogue
  int units, full;
  float* ws;
  unsigned* flags;
  unsigned epoch;
  void* D2;                // EPI_SWIGLU_FWD: act [M, N] bf16, pitch ldd2
  long long ldd2;
  int kb2;                 // k-blocks of the second K segment (0: none)
  int nsplit;              // units beyond `full` are N halves (256 x PBN/2) instead of K halves
  // grouped (MoE expert) GEMM, single-CTA kernel: rows [g_off[e], g_off[e+1])
  // of A and D belong to expert e, whose B is the e-th block of g_bstride rows
  // of the B map (N rows K-major, K rows MN-major); g_off lives on the device
  const int* g_off;
  int g_num;
  int g_bstride;
};
constexpr int MAX_GROUPS = 256;

// Tile -> (first row, first column, expert, end row) of the single-CTA kernel.
// Plain: M fastest. Grouped: expert e owns tiles [tstart[e], tstart[e+1]),
// M fastest within the expert.
struct TileCoord {
  int m0, n0, e, row_end;
};
__device__ __forceinline__ TileCoord tile_coord(const Params& p, const int* tstart, int tile,
                                                int m_tiles, int bm, int bn) {
  TileCoord t;
  if (!p.g_off) {
    t.m0 = (tile % m_tiles) * bm;
    t.n0 = (tile / m_tiles) * bn;
    t.e = 0;
    t.row_end = p.M;
    return t;
  }
  int lo = 0, hi = p.g_num;  // last e with tstart[e] <= tile
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tstart[mid] <= tile) lo = mid; else hi = mid;
  }
  const int r0 = p.g_off[lo], r1 = p.g_off[lo + 1];
  const int mt = (r1 - r0 + bm - 1) / bm, local = tile - tstart[lo];
  t.m0 = r0 + (local % mt) * bm;
  t.n0 = (local / mt) * bn;
  t.e = lo;
  t.row_end = r1;
  return t;
}

// TMA maps of the SwiGLU-backward epilogue: g / u halves of gu and dg / du
// halves of dgu, each [M, N] bf16 with a {32, 32} SWIZZLE_64B box
struct EpiMaps {
  CUtensorMap g, u, dg, du;
  CUtensorMap a2, b2;  // second K segment (pair kernel): D = A B^T + A2 B2^T
  CUtensorMap bh;      // K-major B with PBN/4-row boxes: N-half units of the last wave
};

// Store one 32-column TMEM chunk of a tile row (bf16 [+ residual] / fp32 [+=]).
template <int EPI>
__device__ __forceinline__ void epi_chunk(const Params& p, int row, bool row_ok, int col0_,
                                          const uint32_t (&v)[32]) {
        const int col0 = col0_;
        if (p.trans) {  // D^T of a swapped skinny GEMM: per column, the warp's 32 rows are contiguous
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; ++i) if (col0 + i < p.N) {
              const long long o = (long long)(col0 + i) * p.ldd + row;
              const float f = __uint_as_float(v[i]);
              if (EPI == EPI_BF16) {
                reinterpret_cast<__nv_bfloat16*>(p.D)[o] = __float2bfloat16_rn(f);
              } else {
                float* d = reinterpret_cast<float*>(p.D) + o;
                *d = (EPI == EPI_F32_ACC ? *d : 0.f) + f;
              }
            }
          }
          return;
        }
        if (row_ok && col0 < p.N) {
        const bool full_chunk = p.vec && col0 + 32 <= p.N;
        if (EPI == EPI_SWIGLU_BWD) {
          // same arithmetic as swiglu_bwd_kernel on a bf16-rounded dact, so the
          // fused and the two-kernel paths agree
          const __nv_bfloat16* gr = p.R + (long long)row * p.ldr + col0;
          const __nv_bfloat16* ur = gr + p.N;
          __nv_bfloat16* dg = reinterpret_cast<__nv_bfloat16*>(p.D) + (long long)row * p.ldd + col0;
          __nv_bfloat16* du = dg + p.N;
          auto one = [](float acc, float g, float u, float& og, float& ou) {
            swiglu_bwd_elem(__bfloat162float(__float2bfloat16_rn(acc)), g, u, og, ou);
          };
          if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              const uint4 gv = *reinterpret_cast<const uint4*>(gr + i);
              const uint4 uv = *reinterpret_cast<const uint4*>(ur + i);
              const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&gv);
              const __nv_bfloat16* ub = reinterpret_cast<const __nv_bfloat16*>(&uv);
              float og[8], ou[8];
#pragma unroll
              for (int j = 0; j < 8; ++j)
                one(__uint_as_float(v[i + j]), __bfloat162float(gb[j]), __bfloat162float(ub[j]),
                    og[j], ou[j]);
              *reinterpret_cast<uint4*>(dg + i) =
                  make_uint4(pack_bf16x2(og[0], og[1]), pack_bf16x2(og[2], og[3]),
                             pack_bf16x2(og[4], og[5]), pack_bf16x2(og[6], og[7]));
              *reinterpret_cast<uint4*>(du + i) =
                  make_uint4(pack_bf16x2(ou[0], ou[1]), pack_bf16x2(ou[2], ou[3]),
                             pack_bf16x2(ou[4], ou[5]), pack_bf16x2(ou[6], ou[7]));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) if (col0 + i < p.N) {
              float og, ou;
              one(__uint_as_float(v[i]), __bfloat162float(gr[i]), __bfloat162float(ur[i]), og, ou);
              dg[i] = __float2bfloat16_rn(og);
              du[i] = __float2bfloat16_rn(ou);
            }
          }
        } else if (EPI == EPI_BF16) {
          __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(p.D) + (long long)row * p.ldd + col0;
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
          if (p.R) {
            const __nv_bfloat16* r = p.R + (long long)row * p.ldr + col0;
            if (full_chunk) {
#pragma unroll
              for (int i = 0; i < 32; i += 8) {
                uint4 rv = *reinterpret_cast<const uint4*>(r + i);
                const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&rv);
#pragma unroll
                for (int j = 0; j < 8; ++j) f[i + j] += __bfloat162float(rb[j]);
              }
            } else {
  #pragma unroll
              for (int i = 0; i < 32; ++i) if (col0 + i < p.N) f[i] += __bfloat162float(r[i]);
            }
          }
          if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 o;
              o.x = pack_bf16x2(f[i], f[i + 1]);
              o.y = pack_bf16x2(f[i + 2], f[i + 3]);
              o.z = pack_bf16x2(f[i + 4], f[i + 5]);
              o.w = pack_bf16x2(f[i + 6], f[i + 7]);
              *reinterpret_cast<uint4*>(d + i) = o;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) if (col0 + i < p.N) d[i] = __float2bfloat16_rn(f[i]);
          }
        } else {
          float* d = reinterpret_cast<float*>(p.D) + (long long)row * p.ldd + col0;
          if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float4 o = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                     __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
              if (EPI == EPI_F32_ACC) {
                const float4 old = *reinterpret_cast<const float4*>(d + i);
                o.x += old.x; o.y += old.y; o.z += old.z; o.w += old.w;
              }
              *reinterpret_cast<float4*>(d + i) = o;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) if (col0 + i < p.N)
              d[i] = (EPI == EPI_F32_ACC ? d[i] : 0.f) + __uint_as_float(v[i]);
          }
        }
        }
}

// Single-CTA kernel geometry. TBN = 256 is the general tile; TBN = 32 serves
// the skinny GEMMs of LoRA adapters (one of M / N is the rank): a 128 x 32
// tile keeps every MMA column useful and deepens the ring so one CTA streams
// its long K fast enough (the big operand is read once, HBM-bound).
template <int TBN, int B_MN>
struct SingleCfg {
  static constexpr int B_ROWS = B_MN && TBN < 64 ? 64 : TBN;  // MN-major boxes are 64 wide
  static constexpr int STAGE = A_STAGE_BYTES + B_ROWS * BK * 2;
  static constexpr int STAGES = TBN == 256 ? 4 : 8;
  static constexpr int TMEM = TBN == 256 ? 512 : 64;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static_assert(SMEM <= 232448, "single-CTA GEMM shared memory");
};

template <int A_MN, int B_MN, int EPI, int TBN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma_a,
                const __grid_constant__ CUtensorMap tma_b, Params p) {
  griddep_wait();  // PDL: p.g_off (grouped GEMM) is written by the previous kernel
  using Cfg = SingleCfg<TBN, B_MN>;
  constexpr int BN = TBN, STAGES = Cfg::STAGES, STAGE_BYTES = Cfg::STAGE, TMEM_COLS = Cfg::TMEM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;   // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m_tiles = (p.M + BM - 1) / BM, n_tiles = (p.N + BN - 1) / BN;
  const int k_blocks = (p.K + BK - 1) / BK;
  __shared__ int tstart[MAX_GROUPS + 1];  // grouped: first tile of each expert
  int num_tiles = m_tiles * n_tiles;
  if (p.g_off) {
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int e = 0; e < p.g_num; ++e) {
        tstart[e] = acc;
        acc += (p.g_off[e + 1] - p.g_off[e] + BM - 1) / BM * n_tiles;
      }
      tstart[p.g_num] = acc;
    }
    __syncthreads();
    num_tiles = tstart[p.g_num];
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma_a);
    tma_prefetch(&tma_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  griddep_launch_dependents();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const TileCoord tc = tile_coord(p, tstart, tile, m_tiles, BM, BN);
      const int m0 = tc.m0, n0 = tc.n0;
      const int boff = tc.e * p.g_bstride;  // grouped: this expert's block of B
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * STAGE_BYTES;
        uint8_t* sb = sa + A_STAGE_BYTES;
        mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
        const int k0 = kb * BK;
        if (A_MN) {
          tma_load_2d(sa, &tma_a, &full[stage], m0, k0);
          tma_load_2d(sa + 8192, &tma_a, &full[stage], m0 + 64, k0);
        } else {
          tma_load_2d(sa, &tma_a, &full[stage], k0, m0);
        }
        if (B_MN) {
#pragma unroll
          for (int j = 0; j < Cfg::B_ROWS / 64; ++j)
            tma_load_2d(sb + j * 8192, &tma_b, &full[stage], n0 + 64 * j, boff + k0);
        } else {
          tma_load_2d(sb, &tma_b, &full[stage], k0, boff + n0);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      mbar_wait(&acc_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
        const uint32_t b_addr = a_addr + A_STAGE_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t ad = A_MN ? umma_desc_sw128(a_addr + kk * 2048, 8192, 1024)
                                   : umma_desc_sw128(a_addr + kk * 32, 16, 1024);
          const uint64_t bd = B_MN ? umma_desc_sw128(b_addr + kk * 2048, 8192, 1024)
                                   : umma_desc_sw128(b_addr + kk * 32, 16, 1024);
          umma_f16(d_tmem, ad, bd, idesc, (kb | kk) != 0);
        }
        umma_commit(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      umma_commit(&acc_full[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lane quarter of this warp
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const TileCoord tc = tile_coord(p, tstart, tile, m_tiles, BM, BN);
      const int m0 = tc.m0, n0 = tc.n0;
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < tc.row_end;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * BN + c, v);
        tmem_ld_wait();
        epi_chunk<EPI>(p, row, row_ok, n0 + c, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

// ---- 2-CTA (cta_group::2) variant ---------------------------------------------------
// A CTA pair (cluster of 2 on one TPC) computes a 256x256 tile: CTA r loads
// A rows [128r, 128r+128) and B columns [128r, 128r+128) of the tile (32 KB
// per 64-deep stage instead of 48 KB), the leader issues
// tcgen05.mma.cta_group::2 M256 N256 K16 reading both CTAs' shared memory,
// and each CTA's TMEM receives its 128 rows. Both CTAs' TMA loads complete on
// the leader's full barrier; MMA commits multicast to both CTAs' barriers;
// epilogue warps of both CTAs release the accumulator on the leader's barrier.
// Tile N is 256 (PBN).
constexpr int P_A_BYTES = 128 * BK * 2;     // 16 KB (this CTA's 128 rows of A)
// fp32 epilogue staging for TMA store / reduce-add: per epilogue warp two
// 32 x 32 fp32 chunks (SWIZZLE_128B rows of 128 B)
constexpr int P_EPI_BYTES = 4 * 2 * 32 * 32 * 4;  // 32 KB
template <int PBN, int EPI_>
struct PairCfg {
  // epilogues that store straight from registers (bf16, dual SwiGLU) need no
  // staging buffer: its 32 KB becomes one more operand stage
  static constexpr bool STAGED = EPI_ != 0 && EPI_ != 4;
  static constexpr int B_BYTES = (PBN / 2) * BK * 2;       // this CTA's half of B
  static constexpr int STAGE = P_A_BYTES + B_BYTES;
  static constexpr int EPI_BYTES = STAGED ? P_EPI_BYTES : 0;
  static constexpr int STAGES = (PBN == 256 ? 6 : 8) + (STAGED ? 0 : (PBN == 256 ? 1 : 1));
  static constexpr int SMEM = STAGES * STAGE + EPI_BYTES + 1024 + 256;
  static_assert(SMEM <= 232448, "pair GEMM shared memory");
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int32_t c0, int32_t c1) {
  // completes on the LEADER CTA's barrier (peer bit cleared)
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {  // arrive on both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {  // remote arrive on CTA 0
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, 0;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// fp32 tile chunk smem -> global through the TMA: plain store, or an L2-side
// add (cp.reduce.async.bulk .add.f32) for the accumulate epilogue, so the
// epilogue never waits on a global load of the old value.
template <bool ADD>
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0,
                                             int32_t c1) {
  if (ADD)
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::
            "l"(reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(smem_u32(src)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int A_MN, int B_MN, int EPI, int PBN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tma_a,
                     const __grid_constant__ CUtensorMap tma_b,
                     const __grid_constant__ CUtensorMap tma_d,
                     const __grid_constant__ EpiMaps em, Params p, int n_fastest) {
  using Cfg = PairCfg<PBN, EPI>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + Cfg::STAGES * Cfg::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + Cfg::EPI_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* acc_full = empty + Cfg::STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2] (leader's copy is the one used)
  uint64_t* sw_bar = acc_empty + 2;       // [4 warps x 2] SwiGLU epilogue loads
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(sw_bar + 8);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr bool DUAL = EPI == EPI_SWIGLU_FWD;
  constexpr int TN = DUAL ? PBN / 2 : PBN;  // output columns per tile
  const int m_tiles = (p.M + 255) / 256, n_tiles = (p.N + TN - 1) / TN;
  const int num_tiles = m_tiles * n_tiles;
  const int kb_main = (p.K + BK - 1) / BK;  // segment 1; segment 2 follows
  const int k_blocks = kb_main + p.kb2;
  auto tile_mn = [&](int tile, int& m0, int& n0) {
    const int mt = n_fastest ? tile / n_tiles : tile % m_tiles;
    const int nt = n_fastest ? tile % n_tiles : tile / m_tiles;
    m0 = mt * 256;
    n0 = nt * TN;
  };
  // work unit -> (tile, k-block range, K half: -1 whole, 0 first, 1 second,
  // N half: -1 whole, 0 / 1 = columns [0, PBN/2) / [PBN/2, PBN) of the tile).
  // The last partial wave is split in two along K (long K) or along N.
  int nh_ = -1;
  auto unit_info = [&](int u, int& tile, int& kb0, int& kb1, int& khalf) {
    nh_ = -1;
    if (u < p.full) {
      tile = u, kb0 = 0, kb1 = k_blocks, khalf = -1;
    } else if (p.nsplit) {
      tile = p.full + ((u - p.full) >> 1);
      nh_ = (u - p.full) & 1;
      kb0 = 0, kb1 = k_blocks, khalf = -1;
    } else {
      const int mid = k_blocks / 2;
      tile = p.full + ((u - p.full) >> 1);
      khalf = (u - p.full) & 1;
      kb0 = khalf ? mid : 0;
      kb1 = khalf ? k_blocks : mid;
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tma_a);
    tma_prefetch(&tma_b);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    for (int b = 0; b < 8; ++b) mbar_init(&sw_bar[b], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  // PDL: the prologue above overlapped the previous kernel's tail; nothing of
  // its output is read before this
  griddep_wait();
  griddep_launch_dependents();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs; each loads its halves) ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int u = pair; u < p.units; u += npairs) {
      int tile, kb0, kb1, khalf, m0, n0;
      unit_info(u, tile, kb0, kb1, khalf);
      tile_mn(tile, m0, n0);
      const bool half = nh_ >= 0;  // N-half unit: each CTA loads PBN/4 rows of B
      if (half) n0 += nh_ * (PBN / 2);
      const int am = m0 + 128 * rank;
      const int bn = DUAL ? n0 + (int)rank * p.N : n0 + (half ? PBN / 4 : PBN / 2) * rank;
      const uint32_t stage_tx = half ? Cfg::STAGE - Cfg::B_BYTES / 2 : Cfg::STAGE;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * Cfg::STAGE;
        uint8_t* sb = sa + P_A_BYTES;
        if (leader) mbar_arrive_expect_tx(&full[stage], 2 * stage_tx);
        const bool seg2 = kb >= kb_main;  // LoRA: [X | U] . [W | B]^T without a concat
        const int k0 = (seg2 ? kb - kb_main : kb) * BK;
        // every TMA names its tensor map directly: selecting between
        // __grid_constant__ maps through a pointer makes the compiler copy
        // them to the stack (measured: gate/up fwd 92.6 -> 83.7 % tensor-active)
        auto load_a = [&](const CUtensorMap* m) {
          if (A_MN) {
            tma_load_2d_pair(sa, m, &full[stage], am, k0);
            tma_load_2d_pair(sa + 8192, m, &full[stage], am + 64, k0);
          } else {
            tma_load_2d_pair(sa, m, &full[stage], k0, am);
          }
        };
        auto load_b = [&](const CUtensorMap* m) {
          if (B_MN) {
            tma_load_2d_pair(sb, m, &full[stage], bn, k0);
            if (PBN == 256 && !half) tma_load_2d_pair(sb + 8192, m, &full[stage], bn + 64, k0);
          } else {
            tma_load_2d_pair(sb, m, &full[stage], k0, bn);
          }
        };
        if (!seg2) {
          load_a(&tma_a);
          if (B_MN || !half) load_b(&tma_b);
          else load_b(&em.bh);
        } else {
          load_a(&em.a2);
          load_b(&em.b2);
        }
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (leader only) ----------------
    constexpr uint32_t idesc_full = umma_idesc_bf16(256, PBN, A_MN, B_MN);
    constexpr uint32_t idesc_half = umma_idesc_bf16(256, PBN / 2, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < p.units; u += npairs) {
      int tile, kb0, kb1, khalf;
      unit_info(u, tile, kb0, kb1, khalf);
      const uint32_t idesc = nh_ >= 0 ? idesc_half : idesc_full;
      mbar_wait(&acc_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * PBN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + stage * Cfg::STAGE);
        const uint32_t b_addr = a_addr + P_A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t ad = A_MN ? umma_desc_sw128(a_addr + kk * 2048, 8192, 1024)
                                   : umma_desc_sw128(a_addr + kk * 32, 16, 1024);
          const uint64_t bd = B_MN ? umma_desc_sw128(b_addr + kk * 2048, 8192, 1024)
                                   : umma_desc_sw128(b_addr + kk * 32, 16, 1024);
          umma_f16_pair(d_tmem, ad, bd, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
        }
        umma_commit_pair(&empty[stage]);
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
      }
      umma_commit_pair(&acc_full[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs, 128 rows each) ----------------
    const int q = warp & 3;
    uint32_t epi_chunk_no = 0;  // fp32 TMA epilogue: chunks issued by this warp
    // SwiGLU epilogue: g/u chunks TMA-loaded into two per-warp buffers
    // (g 2 KB | u 2 KB, SWIZZLE_64B rows of 64 B), the next chunk's load in
    // flight while this one is computed; results overwrite the buffer in place
    // and leave through TMA stores
    uint32_t sw_ld = 0, sw_cs = 0;
    uint8_t* sw_buf = epi_smem + q * 8192;
    auto sw_issue = [&](int col, int row) {
      if (lane == 0) {
        const int b = sw_ld & 1;
        bulk_wait_read<0>();  // the store that last read this buffer
        mbar_arrive_expect_tx(&sw_bar[q * 2 + b], 4096);
        tma_load_2d(sw_buf + b * 4096, &em.g, &sw_bar[q * 2 + b], col, row);
        tma_load_2d(sw_buf + b * 4096 + 2048, &em.u, &sw_bar[q * 2 + b], col, row);
      }
      ++sw_ld;
    };
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < p.units; u += npairs) {
      int tile, kb0, kb1, khalf, m0, n0;
      unit_info(u, tile, kb0, kb1, khalf);
      tile_mn(tile, m0, n0);
      const int cw = nh_ >= 0 ? PBN / 2 : PBN;  // accumulator columns of this unit
      if (nh_ >= 0) n0 += nh_ * (PBN / 2);
      const bool sw_tma = EPI == EPI_SWIGLU_BWD && p.tma_swiglu && khalf != 0 &&
                          m0 + 128 * (int)rank + q * 32 < p.M;
      if (sw_tma) {  // needs no accumulator: start before the mainloop finishes
        const int r0 = m0 + 128 * rank + q * 32;
        sw_issue(n0, r0);
        // the rest of the tile's g/u into L2, so each chunk's smem load is an
        // L2 hit rather than a DRAM round trip (one chunk of smem look-ahead)
        if (lane == 0)
          for (int c = 32; c < min(PBN, p.N - n0); c += 32) {
            tma_prefetch_l2(&em.g, n0 + c, r0);
            tma_prefetch_l2(&em.u, n0 + c, r0);
          }
      }
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      const int row0 = m0 + 128 * rank + q * 32;
      const int row = row0 + lane;
      const bool row_ok = row < p.M;
      // split-K: this warp's 32 x PBN slab of the partial in the workspace
      const int slab = ((tile - p.full) * 2 + (int)rank) * 4 + q;
      float* part = khalf >= 0 ? p.ws + (long long)slab * 32 * PBN + lane * PBN : nullptr;
      if (khalf == 0) {  // park the first K half's partial, then raise the flag
#pragma unroll 1
        for (int c = 0; c < PBN; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * PBN + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<uint4*>(part + c + i) = make_uint4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0)
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.flags + slab), "r"(p.epoch)
                       : "memory");
      } else if (khalf == 1) {  // wait for the first half's partial
        unsigned f = 0;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(p.flags + slab) : "memory");
        } while (f != p.epoch);
      }
      auto add_part = [&](int c, uint32_t (&v)[32]) {
        if (khalf != 1) return;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 o = *reinterpret_cast<const float4*>(part + c + i);
          v[i] = __float_as_uint(__uint_as_float(v[i]) + o.x);
          v[i + 1] = __float_as_uint(__uint_as_float(v[i + 1]) + o.y);
          v[i + 2] = __float_as_uint(__uint_as_float(v[i + 2]) + o.z);
          v[i + 3] = __float_as_uint(__uint_as_float(v[i + 3]) + o.w);
        }
      };
      if (khalf == 0) {
        // nothing to store: the partial is parked
      } else if (EPI == EPI_SWIGLU_BWD && p.tma_swiglu) {
        const int c_end = sw_tma ? min(PBN, p.N - n0) : 0;
#pragma unroll 1
        for (int c = 0; c < c_end; c += 32) {
          if (c + 32 < c_end) sw_issue(n0 + c + 32, row0);
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * PBN + c, v);
          tmem_ld_wait();
          add_part(c, v);
          const int b = sw_cs & 1;
          mbar_wait(&sw_bar[q * 2 + b], (sw_cs >> 1) & 1);
          ++sw_cs;
          uint8_t* gb = sw_buf + b * 4096;
          uint8_t* ub = gb + 2048;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int off = lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4);
            const uint4 gv = *reinterpret_cast<const uint4*>(gb + off);
            const uint4 uv = *reinterpret_cast<const uint4*>(ub + off);
            const __nv_bfloat16* g8 = reinterpret_cast<const __nv_bfloat16*>(&gv);
            const __nv_bfloat16* u8 = reinterpret_cast<const __nv_bfloat16*>(&uv);
            float og[8], ou[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              swiglu_bwd_elem(__bfloat162float(__float2bfloat16_rn(__uint_as_float(v[8 * k + j]))),
                              __bfloat162float(g8[j]), __bfloat162float(u8[j]), og[j], ou[j]);
            }
            *reinterpret_cast<uint4*>(gb + off) =
                make_uint4(pack_bf16x2(og[0], og[1]), pack_bf16x2(og[2], og[3]),
                           pack_bf16x2(og[4], og[5]), pack_bf16x2(og[6], og[7]));
            *reinterpret_cast<uint4*>(ub + off) =
                make_uint4(pack_bf16x2(ou[0], ou[1]), pack_bf16x2(ou[2], ou[3]),
                           pack_bf16x2(ou[4], ou[5]), pack_bf16x2(ou[6], ou[7]));
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d<false>(&em.dg, gb, n0 + c, row0);
            tma_store_2d<false>(&em.du, ub, n0 + c, row0);
            bulk_commit();
          }
        }
      } else if (EPI == EPI_SWIGLU_FWD) {
        const int c_end = min(TN, p.N - n0);
#pragma unroll 1
        for (int c = 0; c < c_end; c += 32) {
          uint32_t vg[32], vu[32];
          tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * PBN + c, vg);
          tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * PBN + TN + c, vu);
          tmem_ld_wait();
          if (row_ok) {
            __nv_bfloat16* dg = reinterpret_cast<__nv_bfloat16*>(p.D) + (long long)row * p.ldd + n0 + c;
            __nv_bfloat16* du = dg + p.N;
            __nv_bfloat16* da = reinterpret_cast<__nv_bfloat16*>(p.D2) + (long long)row * p.ldd2 + n0 + c;
            if (p.vec && n0 + c + 32 <= p.N) {
#pragma unroll
              for (int i = 0; i < 32; i += 8) {
                uint32_t pg[4], pu[4], pa[4];
#pragma unroll
                for (int j = 0; j < 8; j += 2) {
                  pg[j / 2] = pack_bf16x2(__uint_as_float(vg[i + j]), __uint_as_float(vg[i + j + 1]));
                  pu[j / 2] = pack_bf16x2(__uint_as_float(vu[i + j]), __uint_as_float(vu[i + j + 1]));
                  // act from the bf16-rounded g, u: what the two-kernel path reads back
                  const __nv_bfloat162 g2 = *reinterpret_cast<const __nv_bfloat162*>(&pg[j / 2]);
                  const __nv_bfloat162 u2 = *reinterpret_cast<const __nv_bfloat162*>(&pu[j / 2]);
                  pa[j / 2] = pack_bf16x2(
                      swiglu_fwd_elem(__bfloat162float(g2.x), __bfloat162float(u2.x)),
                      swiglu_fwd_elem(__bfloat162float(g2.y), __bfloat162float(u2.y)));
                }
                *reinterpret_cast<uint4*>(dg + i) = make_uint4(pg[0], pg[1], pg[2], pg[3]);
                *reinterpret_cast<uint4*>(du + i) = make_uint4(pu[0], pu[1], pu[2], pu[3]);
                *reinterpret_cast<uint4*>(da + i) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
              }
            } else {
  #pragma unroll
              for (int i = 0; i < 32; ++i) if (n0 + c + i < p.N) {
                const __nv_bfloat16 g = __float2bfloat16_rn(__uint_as_float(vg[i]));
                const __nv_bfloat16 u = __float2bfloat16_rn(__uint_as_float(vu[i]));
                dg[i] = g;
                du[i] = u;
                da[i] = __float2bfloat16_rn(swiglu_fwd_elem(__bfloat162float(g), __bfloat162float(u)));
              }
            }
          }
        }
      } else if ((EPI == EPI_F32 || EPI == EPI_F32_ACC) && p.tma_out) {
        // fp32: 32x32 chunks through swizzled smem and the TMA (store or L2 add),
        // two chunk buffers per warp in flight
        uint8_t* wbuf = epi_smem + q * (2 * 4096);
        // chunks wholly outside D are skipped (warp-uniform), so every written
        // buffer belongs to a committed store and "two chunks ago" holds
        const int c_end = min(cw, p.N - n0);
#pragma unroll 1
        for (int c = 0; c < c_end && row0 < p.M; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * PBN + c, v);
          tmem_ld_wait();
          add_part(c, v);
          uint8_t* buf = wbuf + (epi_chunk_no++ & 1) * 4096;  // alternates across tiles too
          if (lane == 0) bulk_wait_read<1>();  // the store from this buffer two chunks ago
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(buf + lane * 128 + ((k ^ (lane & 7)) << 4)) =
                make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d<EPI == EPI_F32_ACC>(&tma_d, buf, n0 + c, row0);
            bulk_commit();
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < cw; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * PBN + c, v);
          tmem_ld_wait();
          add_part(c, v);
          epi_chunk<EPI>(p, row, row_ok, n0 + c, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&acc_empty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (((EPI != EPI_BF16 && p.tma_out) || (EPI == EPI_SWIGLU_BWD && p.tma_swiglu)) && lane == 0)
      bulk_wait_all();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
}

// ---- host side: tensor maps ------------------------------------------------------

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

// 2-D bf16 map over a row-major [rows, cols] matrix (cols contiguous, row
// pitch ld elements) with a {box_cols, box_rows} SWIZZLE_128B box.
bool make_map(CUtensorMap* map, const void* base, long long rows, long long cols, long long ld,
              int box_cols, int box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t elem[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
            box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// fp32 [rows, cols] (row pitch ld elements), box {32 cols, 32 rows}, SWIZZLE_128B:
// the epilogue's TMA store / reduce-add target
bool make_map_f32(CUtensorMap* map, const void* base, long long rows, long long cols,
                  long long ld) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t elem[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
            elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// bf16 [rows, cols] (row pitch ld elements), box {32 cols, 32 rows}, SWIZZLE_64B:
// the SwiGLU-backward epilogue's g/u loads and dg/du stores
bool make_map_sw64(CUtensorMap* map, const void* base, long long rows, long long cols,
                   long long ld) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t elem[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Split-K scratch per stream (GEMMs on the compute and weight-gradient
// streams may run concurrently): fp32 partial slabs + per-warp flags that
// carry a launch epoch, so they never need resetting.
struct SplitWs {
  float* ws = nullptr;
  unsigned* flags = nullptr;
  unsigned epoch = 0;
};
SplitWs split_ws(cudaStream_t st, std::size_t elems, std::size_t flags) {
  Workspace* a = stream_workspace(st, WS_SPLITK_PARTIALS,
                                  4 * std::max<std::size_t>(elems, (std::size_t)37 * 2 * 128 * 256));
  Workspace* f = stream_workspace(st, WS_SPLITK_FLAGS, 4 * std::max<std::size_t>(flags, 37 * 8));
  if (!a || !f) return SplitWs{};
  return SplitWs{static_cast<float*>(a->p), static_cast<unsigned*>(f->p), ++f->epoch};
}

// Pair tiles are 256 x 256 (256 x 128 pair tiles would fill the 74 pairs'
// last wave better for 4096-wide GEMMs, but measured ~1.0 PF/s vs ~1.35 on
// B200: half-size MMAs double the per-k-block pipeline overhead).
constexpr int PBN = 256;

// Launch with programmatic stream serialization (PDL): the grid may be
// scheduled while the stream's previous kernel drains, its CTAs run their
// prologue (barriers, TMEM allocation, tensor-map prefetch) and then block in
// griddep_wait() until that kernel has completed. The GEMMs trigger their own
// dependents right after their prologue.
template <class K, class... Args>
cudaError_t launch_pdl(K kern, dim3 grid, int smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t c = {};
  c.gridDim = grid;
  c.blockDim = dim3(NUM_THREADS, 1, 1);
  c.dynamicSmemBytes = smem;
  c.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = at;
  c.numAttrs = 1;
  return cudaLaunchKernelEx(&c, kern, args...);
}

// why the last rp_gemm_* call on this thread failed (rp_gemm_last_error)
thread_local const char* g_gemm_why = "";
inline cudaError_t launch_status(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) g_gemm_why = what;
  return e;
}

template <int A_MN, int B_MN, int EPI>
cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& td,
                   const EpiMaps& em, const Params& p, bool pair, int n_fastest,
                   cudaStream_t stream) {
  if (pair) {
    auto kern = gemm_pair_kernel<A_MN, B_MN, EPI, PBN>;
    const int smem = PairCfg<PBN, EPI>::SMEM;
    if (!ensure_smem_t(kern, smem)) return g_gemm_why = "pair kernel: shared-memory attribute", cudaErrorInvalidValue;
    const int pbn = PBN;
    const int tn = EPI == EPI_SWIGLU_FWD ? pbn / 2 : pbn;  // output columns per tile
    const int tiles = ((p.M + 255) / 256) * ((p.N + tn - 1) / tn);
    const int npairs = num_sms() / 2;
    Params q = p;
    q.units = q.full = tiles;
    // split-K of a short last wave: its tiles become two K halves each, so
    // the wave finishes in about half the time. Only for long K (>= 8192):
    // measured +6 % on 4096x4096x12288 and 4096x4096x24576, but -2..-5 % at
    // K = 4096, where parking and re-reading the 128 KB fp32 partial per CTA
    // costs about what the shorter wave saves
    const int full = (tiles / npairs) * npairs, tail = tiles - full;
    // a short last wave at moderate K: its tiles become two 256 x PBN/2 halves
    // (no partials to reduce, unlike the K split); plain epilogues only
    if ((EPI == EPI_BF16 || EPI == EPI_F32 || EPI == EPI_F32_ACC) &&
        q.kb2 == 0 && tail > 0 && 2 * tail <= npairs && p.K < 8192) {
      q.full = full;
      q.units = full + 2 * tail;
      q.nsplit = 1;
    } else if (EPI != EPI_SWIGLU_BWD && EPI != EPI_SWIGLU_FWD && tail > 0 && 2 * tail <= npairs && p.K >= 8192) {
      const SplitWs w = split_ws(stream, (std::size_t)tail * 2 * 128 * pbn, (std::size_t)tail * 8);
      if (w.ws) {
        q.full = full;
        q.units = full + 2 * tail;
        q.ws = w.ws;
        q.flags = w.flags;
        q.epoch = w.epoch;
      }
    }
    const int pairs = q.units < npairs ? q.units : npairs;
    return launch_pdl(kern, dim3(2 * pairs), smem, stream, ta, tb, td, em, q, n_fastest) == cudaSuccess
               ? cudaSuccess
               : launch_status("pair kernel launch");
  }
  const bool skinny = p.N <= 32;
  auto kern = skinny ? gemm_kernel<A_MN, B_MN, EPI, 32> : gemm_kernel<A_MN, B_MN, EPI, 256>;
  const int smem = skinny ? SingleCfg<32, B_MN>::SMEM : SingleCfg<256, B_MN>::SMEM;
  if (!ensure_smem_t(kern, smem)) return g_gemm_why = "single kernel: shared-memory attribute", cudaErrorInvalidValue;
  const int tbn = skinny ? 32 : BN;
  int tiles = ((p.M + BM - 1) / BM) * ((p.N + tbn - 1) / tbn);
  if (p.g_off) tiles += p.g_num * ((p.N + tbn - 1) / tbn);  // ragged last m-tile per group (bound)
  const int grid = tiles < num_sms() ? tiles : num_sms();
  return launch_pdl(kern, dim3(grid), smem, stream, ta, tb, p) == cudaSuccess
             ? cudaSuccess
             : launch_status("single kernel launch");
}

template <int A_MN, int B_MN>
cudaError_t dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb,
                         const CUtensorMap& td, const EpiMaps& em, const Params& p, bool pair,
                         int n_fastest, cudaStream_t s) {
  switch (epi) {
    case EPI_BF16: return launch<A_MN, B_MN, EPI_BF16>(ta, tb, td, em, p, pair, n_fastest, s);
    case EPI_F32: return launch<A_MN, B_MN, EPI_F32>(ta, tb, td, em, p, pair, n_fastest, s);
    case EPI_SWIGLU_FWD:  // pair kernel, gate/up forward layout only
      if constexpr (A_MN == 0 && B_MN == 0) {
        if (!pair) return g_gemm_why = "SwiGLU forward epilogue needs pair tiles", cudaErrorInvalidValue;
        return launch<A_MN, B_MN, EPI_SWIGLU_FWD>(ta, tb, td, em, p, pair, n_fastest, s);
      } else {
        return g_gemm_why = "SwiGLU forward epilogue: K-major operands only", cudaErrorInvalidValue;
      }
    case EPI_SWIGLU_BWD:  // only the down-projection dgrad layout is instantiated
      if constexpr (A_MN == 0 && B_MN == 1)
        return launch<A_MN, B_MN, EPI_SWIGLU_BWD>(ta, tb, td, em, p, pair, n_fastest, s);
      else
        return g_gemm_why = "SwiGLU backward epilogue: A K-major, B MN-major only", cudaErrorInvalidValue;
    default: return launch<A_MN, B_MN, EPI_F32_ACC>(ta, tb, td, em, p, pair, n_fastest, s);
  }
}

}  // namespace
}  // namespace rp

using namespace rp;

// mode 0: plain GEMM; 1: SwiGLU-backward epilogue; 2: dual gate/up forward
// with the SwiGLU epilogue (act, ld_act)
struct Seg2 {
  const void* A2 = nullptr;
  long long lda2 = 0;
  const void* B2 = nullptr;
  long long ldb2 = 0;
  int K2 = 0;
};

static int gemm_entry(const rp_gemm_args_t* g, void* stream, int mode, void* act = nullptr,
                      long long ld_act = 0, const Seg2& s2 = Seg2()) {
  const bool swiglu_bwd = mode == 1, dual = mode == 2;
  // M <= 32 (e.g. a LoRA A-gradient, M = rank): compute D^T = B A^T with the
  // roles swapped — its N is the small side, served by 128 x 32 tiles — and
  // store it transposed
  bool trans = false;
  rp_gemm_args_t sw;
  if (mode == 0 && g && g->M <= 32 && g->N > 32 && !g->R && !s2.K2) {
    sw = *g;
    sw.M = g->N;
    sw.N = g->M;
    sw.A = g->B;
    sw.lda = g->ldb;
    sw.a_mn_major = g->b_mn_major;
    sw.B = g->A;
    sw.ldb = g->lda;
    sw.b_mn_major = g->a_mn_major;
    g = &sw;
    trans = true;
  }
  g_gemm_why = "";
  if (!g || g->M <= 0 || g->N <= 0 || g->K <= 0 || !g->A || !g->B || !g->D)
    return g_gemm_why = "bad shape or null operand", RP_E_INPUT;
  if ((g->lda * 2) % 16 || (g->ldb * 2) % 16 || (reinterpret_cast<uintptr_t>(g->A) & 15) ||
      (reinterpret_cast<uintptr_t>(g->B) & 15))
    return RP_E_INPUT;
  // CTA pairs (cta_group::2, 256-row tiles) whenever M fills a pair tile
  // N <= 32 (LoRA rank side): 128 x 32 single-CTA tiles, except few row tiles
  // with a long K, where the pair kernel measured faster (dU = dY B, K = 24576)
  const bool skinny = mode == 0 && g->N <= 32 && !(g->M / 128 < num_sms() && g->K > 8192);
  const bool pair = g->M >= 256 && !skinny;
  CUtensorMap ta, tb;
  bool ok = g->a_mn_major ? make_map(&ta, g->A, g->K, g->M, g->lda, 64, 64)
                          : make_map(&ta, g->A, g->M, g->K, g->lda, 64, BM);
  ok = ok && (g->b_mn_major ? make_map(&tb, g->B, g->K, g->N, g->ldb, 64, 64)
                            : make_map(&tb, g->B, dual ? 2LL * g->N : g->N, g->K, g->ldb, 64,
                                       pair ? PBN / 2
                                            : g->N <= 32 ? 32 : BN));  // = launch()'s tile
  // raster: keep the larger operand's tile hot (walk the other dimension fastest)
  const int n_fastest = (double)g->M > (double)g->N ? 1 : 0;
  if (!ok) return g_gemm_why = "A/B tensor map encode", RP_E_CUDA;
  const int esz = g->out_f32 ? 4 : 2;
  const bool vec = (g->ldd * esz) % 16 == 0 && (reinterpret_cast<uintptr_t>(g->D) & 15) == 0 &&
                   (!g->R || ((g->ldr * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(g->R) & 15) == 0)) &&
                   (!dual || ((ld_act * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(act) & 15) == 0 &&
                              g->N % 8 == 0));
  // fp32 outputs of the pair kernel go through a TMA map (store / L2 reduce-add)
  CUtensorMap td;
  std::memset(&td, 0, sizeof(td));
  // (not for a swapped skinny GEMM: its D is stored transposed, element by
  // element in epi_chunk — a TMA map over the swapped shape would write rows
  // of the untransposed layout past the end of D)
  const bool tma_out = pair && !trans && g->out_f32 && (g->ldd * 4) % 16 == 0 &&
                       (reinterpret_cast<uintptr_t>(g->D) & 15) == 0 &&
                       make_map_f32(&td, g->D, g->M, g->N, g->ldd);
  EpiMaps em;
  std::memset(&em, 0, sizeof(em));
  const auto* R16 = reinterpret_cast<const __nv_bfloat16*>(g->R);
  auto* D16 = reinterpret_cast<__nv_bfloat16*>(g->D);
  const bool tma_swiglu = swiglu_bwd && pair && vec &&
                          make_map_sw64(&em.g, R16, g->M, g->N, g->ldr) &&
                          make_map_sw64(&em.u, R16 + g->N, g->M, g->N, g->ldr) &&
                          make_map_sw64(&em.dg, D16, g->M, g->N, g->ldd) &&
                          make_map_sw64(&em.du, D16 + g->N, g->M, g->N, g->ldd);
  if (pair && !g->b_mn_major && !dual &&
      !make_map(&em.bh, g->B, g->N, g->K, g->ldb, 64, PBN / 4))
    return g_gemm_why = "N-half B tensor map encode", RP_E_CUDA;
  if (s2.K2 > 0) {  // second K segment: same majors and boxes as A / B
    if (!pair) return RP_E_INPUT;
    const bool ok2 =
        (g->a_mn_major ? make_map(&em.a2, s2.A2, s2.K2, g->M, s2.lda2, 64, 64)
                       : make_map(&em.a2, s2.A2, g->M, s2.K2, s2.lda2, 64, BM)) &&
        (g->b_mn_major ? make_map(&em.b2, s2.B2, s2.K2, g->N, s2.ldb2, 64, 64)
                       : make_map(&em.b2, s2.B2, dual ? 2LL * g->N : g->N, s2.K2, s2.ldb2, 64,
                                  PBN / 2));
    if (!ok2) return g_gemm_why = "second-segment tensor map encode", RP_E_CUDA;
  }
  Params p{g->M, g->N, g->K, g->D, g->ldd, R16, g->ldr, vec ? 1 : 0, tma_out ? 1 : 0,
           tma_swiglu ? 1 : 0, trans ? 1 : 0, 0, 0,
           nullptr, nullptr, 0, act, ld_act, (s2.K2 + BK - 1) / BK};
  const int epi = dual ? EPI_SWIGLU_FWD : swiglu_bwd ? EPI_SWIGLU_BWD
                             : g->out_f32 ? (g->accumulate ? EPI_F32_ACC : EPI_F32) : EPI_BF16;
  if (g->out_f32 && g->R) return RP_E_INPUT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (g->a_mn_major)
    e = g->b_mn_major ? dispatch_epi<1, 1>(epi, ta, tb, td, em, p, pair, n_fastest, s)
                      : dispatch_epi<1, 0>(epi, ta, tb, td, em, p, pair, n_fastest, s);
  else
    e = g->b_mn_major ? dispatch_epi<0, 1>(epi, ta, tb, td, em, p, pair, n_fastest, s)
                      : dispatch_epi<0, 0>(epi, ta, tb, td, em, p, pair, n_fastest, s);
  return e == cudaSuccess ? RP_OK : RP_E_CUDA;
}

extern "C" __attribute__((visibility("default"))) const char* rp_gemm_last_error(void) {
  return rp::g_gemm_why;
}

extern "C" __attribute__((visibility("default"))) int rp_gemm_bf16(const rp_gemm_args_t* g,
                                                                   void* stream) {
  return gemm_entry(g, stream, 0);
}

extern "C" __attribute__((visibility("default"))) int rp_gemm_swiglu_fwd(const rp_gemm_args_t* g,
                                                                         void* act, int64_t ld_act,
                                                                         void* stream) {
  if (!g || !act || g->out_f32 || g->accumulate || g->R || g->N % 8 || g->a_mn_major ||
      g->b_mn_major)
    return RP_E_INPUT;
  if (g->M >= 256) return gemm_entry(g, stream, 2, act, ld_act);
  // below one pair tile: the plain GEMM into gu, then the SwiGLU kernel
  rp_gemm_args_t a = *g;
  a.N = 2 * g->N;
  const int rc = gemm_entry(&a, stream, 0);
  if (rc != RP_OK || ld_act != g->N || g->ldd != 2LL * g->N) return rc != RP_OK ? rc : RP_E_INPUT;
  return rp_swiglu_fwd(g->D, act, g->M, g->N, stream);
}

extern "C" __attribute__((visibility("default"))) int rp_gemm_swiglu_bwd(const rp_gemm_args_t* g,
                                                                         void* stream) {
  if (!g || g->out_f32 || g->accumulate || !g->R || g->N % 8 || g->a_mn_major || !g->b_mn_major)
    return RP_E_INPUT;
  return gemm_entry(g, stream, 1);
}

// D = A B^T + A2 B2^T (+ R): a second K segment with the same majors, read by
// the producer after A / B's k-blocks — the LoRA up-projection folded into the
// base GEMM without materialising [X | U] or [W | B]. Pair tiles only (M >= 256).
extern "C" __attribute__((visibility("default"))) int rp_gemm_bf16_2seg(
    const rp_gemm_args_t* g, const void* A2, int64_t lda2, const void* B2, int64_t ldb2,
    int32_t K2, void* stream) {
  if (!g || !A2 || !B2 || K2 <= 0 || (lda2 * 2) % 16 || (ldb2 * 2) % 16 ||
      (reinterpret_cast<uintptr_t>(A2) & 15) || (reinterpret_cast<uintptr_t>(B2) & 15))
    return RP_E_INPUT;
  if (g->M < 256 || g->N <= 32) {  // below a pair tile: two GEMMs, the second adds into D
    int rc = gemm_entry(g, stream, 0);
    if (rc != RP_OK) return rc;
    rp_gemm_args_t b = *g;
    b.A = A2;
    b.lda = lda2;
    b.B = B2;
    b.ldb = ldb2;
    b.K = K2;
    if (g->out_f32) {
      b.accumulate = 1;
    } else {
      b.R = g->D;
      b.ldr = g->ldd;
    }
    return gemm_entry(&b, stream, 0);
  }
  Seg2 s2;
  s2.A2 = A2;
  s2.lda2 = lda2;
  s2.B2 = B2;
  s2.ldb2 = ldb2;
  s2.K2 = K2;
  return gemm_entry(g, stream, 0, nullptr, 0, s2);
}

// One entry for every epilogue with an optional second K segment:
// epilogue 0 = rp_gemm_bf16, 1 = rp_gemm_swiglu_bwd, 2 = rp_gemm_swiglu_fwd
// (act / ld_act); K2 > 0 adds A2 . B2^T as in rp_gemm_bf16_2seg. The fused
// SwiGLU epilogues with a second segment need M >= 256 (pair tiles).
extern "C" __attribute__((visibility("default"))) int rp_gemm_ex(
    const rp_gemm_args_t* g, int32_t epilogue, void* act, int64_t ld_act, const void* A2,
    int64_t lda2, const void* B2, int64_t ldb2, int32_t K2, void* stream) {
  if (!g || epilogue < 0 || epilogue > 2) return RP_E_INPUT;
  if (K2 <= 0) {
    if (epilogue == 0) return rp_gemm_bf16(g, stream);
    if (epilogue == 1) return rp_gemm_swiglu_bwd(g, stream);
    return rp_gemm_swiglu_fwd(g, act, ld_act, stream);
  }
  if (epilogue == 0) return rp_gemm_bf16_2seg(g, A2, lda2, B2, ldb2, K2, stream);
  if (g->M < 256 || !A2 || !B2 || (lda2 * 2) % 16 || (ldb2 * 2) % 16 || g->out_f32 ||
      g->accumulate || g->N % 8)
    return RP_E_INPUT;
  if (epilogue == 1 && (!g->R || g->a_mn_major || !g->b_mn_major)) return RP_E_INPUT;
  if (epilogue == 2 && (!act || g->R || g->a_mn_major || g->b_mn_major)) return RP_E_INPUT;
  Seg2 s2;
  s2.A2 = A2;
  s2.lda2 = lda2;
  s2.B2 = B2;
  s2.ldb2 = ldb2;
  s2.K2 = K2;
  return gemm_entry(g, stream, epilogue, act, ld_act, s2);
}

// Grouped (MoE expert) GEMM: rows [row_off[e], row_off[e+1]) of A (K-major,
// args->M rows in all) and D are multiplied by expert e's B — the e-th block
// of b_group_rows rows of B (K-major: [groups*N, K], b_group_rows = N;
// MN-major: [groups*K, N], b_group_rows = K). row_off (groups+1 int32) is a
// DEVICE array, so the routing never syncs the host. epilogue 0: bf16 D
// (+ R); 1: the SwiGLU-backward epilogue (R = gu [M, 2N], D = dgu, B
// MN-major). Single-CTA 128 x 256 tiles, persistent over all experts' tiles.
extern "C" __attribute__((visibility("default"))) int rp_gemm_grouped(
    const rp_gemm_args_t* g, const int32_t* row_off, int32_t groups, int32_t b_group_rows,
    int32_t epilogue, void* stream) {
  if (!g || !row_off || groups <= 0 || groups > MAX_GROUPS || b_group_rows <= 0 ||
      epilogue < 0 || epilogue > 1 || g->M <= 0 || g->N <= 32 || g->K <= 0 || !g->A || !g->B ||
      !g->D || g->a_mn_major || g->out_f32 || g->accumulate)
    return RP_E_INPUT;
  if (epilogue == 1 && (!g->R || !g->b_mn_major || g->N % 8)) return RP_E_INPUT;
  if ((g->lda * 2) % 16 || (g->ldb * 2) % 16 || (reinterpret_cast<uintptr_t>(g->A) & 15) ||
      (reinterpret_cast<uintptr_t>(g->B) & 15))
    return RP_E_INPUT;
  CUtensorMap ta, tb, td;
  std::memset(&td, 0, sizeof(td));
  const long long brows = (long long)groups * b_group_rows;
  bool ok = make_map(&ta, g->A, g->M, g->K, g->lda, 64, BM);
  ok = ok && (g->b_mn_major ? make_map(&tb, g->B, brows, g->N, g->ldb, 64, 64)
                            : make_map(&tb, g->B, brows, g->K, g->ldb, 64, BN));
  if (!ok) return RP_E_CUDA;
  EpiMaps em;
  std::memset(&em, 0, sizeof(em));
  const bool vec = (g->ldd * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(g->D) & 15) == 0 &&
                   (!g->R || ((g->ldr * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(g->R) & 15) == 0));
  Params p{g->M, g->N, g->K, g->D, g->ldd, reinterpret_cast<const __nv_bfloat16*>(g->R), g->ldr,
           vec ? 1 : 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, nullptr, 0, 0, 0,
           row_off, groups, b_group_rows};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (epilogue == 1)
    e = launch<0, 1, EPI_SWIGLU_BWD>(ta, tb, td, em, p, false, 0, s);
  else
    e = g->b_mn_major ? launch<0, 1, EPI_BF16>(ta, tb, td, em, p, false, 0, s)
                      : launch<0, 0, EPI_BF16>(ta, tb, td, em, p, false, 0, s);
  return e == cudaSuccess ? RP_OK : RP_E_CUDA;
}
