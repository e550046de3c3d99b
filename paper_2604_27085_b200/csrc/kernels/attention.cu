// Causal GQA flash attention, forward and backward (head_dim 64 / 128, bf16).
//
// Round-1 implementation on the warp-level tensor-core path
// (mma.sync m16n8k16 bf16 -> f32, ldmatrix from XOR-swizzled shared memory,
// cp.async double buffering). The tcgen05/TMEM port of these two kernels is
// the next step recorded in DESIGN.md; the GEMMs, which carry ~90% of the
// step's FLOPs, are already tcgen05.
//
// Layouts (token-major, as produced by the fused QKV GEMM + QK-norm/RoPE):
//   q [T, nq, hd], k/v [T, nk, hd] (row pitches ldq/ldk/ldv), o like q,
//   lse [nq, T] (natural log). T = batch * seq, sequences packed, causal
//   within a sequence; seq % 128 == 0.
// Forward: block = 128 queries x 1 head (8 warps x 16 rows), K/V tiles of
//   64 keys, online softmax in exp2 domain.
// Backward: block = 64 keys x 1 KV head (4 warps x 16 keys); loops over the
//   G = nq/nk query heads of the group and all later query tiles, keeping
//   dK/dV for its keys in registers; dQ is reduced through fp32 atomics into
//   a workspace and cast at the end. delta = rowsum(dO * O) is a pre-pass.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rp/kernels.h"

namespace rp {
namespace {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Swizzled [rows][W] bf16 tile: 16-byte chunk c of row r lives at c ^ (r & 7).
template <int W>
__device__ __forceinline__ int swz(int r, int c /*element col, multiple of 8*/) {
  return r * W + ((((c >> 3) ^ (r & 7))) << 3);
}

// async copy of a [ROWS][HD] tile (rows from a strided bf16 matrix) into smem
template <int ROWS, int HD, int THREADS>
__device__ __forceinline__ void load_tile(bf16* s, const bf16* g, long long ld) {
  constexpr int CH = HD / 8;
#pragma unroll
  for (int i = threadIdx.x; i < ROWS * CH; i += THREADS) {
    const int r = i / CH, c = (i % CH) * 8;
    cp_async16(s + swz<HD>(r, c), g + (long long)r * ld + c);
  }
}

constexpr float LOG2E = 1.4426950408889634f;

// ------------------------------------------------------------------ forward
template <int HD>
__global__ void __launch_bounds__(256)
    attn_fwd_kernel(const bf16* __restrict__ q, long long ldq, const bf16* __restrict__ k,
                    long long ldk, const bf16* __restrict__ v, long long ldv,
                    bf16* __restrict__ o, long long ldo, float* __restrict__ lse, int T, int seq,
                    int nq, int nk, float scale) {
  constexpr int BM = 128, BN = 64, THREADS = 256, DK = HD / 16, DN = HD / 8;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  bf16* sK = sQ + BM * HD;       // [2][BN][HD]
  bf16* sV = sK + 2 * BN * HD;   // [2][BN][HD]

  const int qblocks = T / BM;
  const int qb = qblocks - 1 - blockIdx.x;  // heaviest (latest) query tiles first
  const int h = blockIdx.y, kvh = h / (nq / nk);
  const int q0 = qb * BM;
  const int s0 = (q0 / seq) * seq;
  const int nkb = (q0 - s0 + BM) / BN;  // key tiles [s0, q0 + BM)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane / 4, qd = lane % 4;

  load_tile<BM, HD, THREADS>(sQ, q + (long long)q0 * ldq + (long long)h * HD, ldq);
  load_tile<BN, HD, THREADS>(sK, k + (long long)s0 * ldk + (long long)kvh * HD, ldk);
  load_tile<BN, HD, THREADS>(sV, v + (long long)s0 * ldv + (long long)kvh * HD, ldv);
  cp_commit();

  float oacc[DN][4];
#pragma unroll
  for (int i = 0; i < DN; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  const float sl2 = scale * LOG2E;
  uint32_t qf[DK][4];
  const int row_base = warp * 16;
  const int qrow0 = q0 + row_base + g, qrow1 = qrow0 + 8;

  for (int kb = 0; kb < nkb; ++kb) {
    cp_wait<0>();
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int ks = 0; ks < DK; ++ks) {
        const int mi = lane / 8, ri = lane % 8;
        ldsm_x4(qf[ks], smem_addr(sQ + swz<HD>(row_base + ri + (mi & 1) * 8, ks * 16 + (mi >> 1) * 8)));
      }
    }
    if (kb + 1 < nkb) {
      const int nb = (kb + 1) & 1;
      const long long key0 = s0 + (long long)(kb + 1) * BN;
      load_tile<BN, HD, THREADS>(sK + nb * BN * HD, k + key0 * ldk + (long long)kvh * HD, ldk);
      load_tile<BN, HD, THREADS>(sV + nb * BN * HD, v + key0 * ldv + (long long)kvh * HD, ldv);
      cp_commit();
    }
    const bf16* tK = sK + (kb & 1) * BN * HD;
    const bf16* tV = sV + (kb & 1) * BN * HD;

    float s[BN / 8][4];
#pragma unroll
    for (int i = 0; i < BN / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < DK; ++ks) {
#pragma unroll
      for (int p = 0; p < BN / 16; ++p) {
        uint32_t b[4];
        const int mi = lane / 8, ri = lane % 8;
        ldsm_x4(b, smem_addr(tK + swz<HD>(p * 16 + ri + (mi >> 1) * 8, ks * 16 + (mi & 1) * 8)));
        mma16816(s[2 * p], qf[ks], b[0], b[1]);
        mma16816(s[2 * p + 1], qf[ks], b[2], b[3]);
      }
    }
    // causal mask on the diagonal tiles
    const int key_base = s0 + kb * BN;
    if (key_base + BN - 1 > q0 + row_base) {
#pragma unroll
      for (int nb = 0; nb < BN / 8; ++nb) {
        const int kc = key_base + nb * 8 + 2 * qd;
        if (kc > qrow0) s[nb][0] = -INFINITY;
        if (kc + 1 > qrow0) s[nb][1] = -INFINITY;
        if (kc > qrow1) s[nb][2] = -INFINITY;
        if (kc + 1 > qrow1) s[nb][3] = -INFINITY;
      }
    }
    // online softmax (two rows per thread: g and g+8)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float mx = -INFINITY;
#pragma unroll
      for (int nb = 0; nb < BN / 8; ++nb) mx = fmaxf(mx, fmaxf(s[nb][2 * r], s[nb][2 * r + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run[r], mx);
      const float corr = m_run[r] == -INFINITY ? 0.f : exp2f((m_run[r] - m_new) * sl2);
      m_run[r] = m_new;
      l_run[r] *= corr;
#pragma unroll
      for (int dn = 0; dn < DN; ++dn) {
        oacc[dn][2 * r] *= corr;
        oacc[dn][2 * r + 1] *= corr;
      }
      const float mb = m_new * sl2;
#pragma unroll
      for (int nb = 0; nb < BN / 8; ++nb) {
        const float p0 = exp2f(s[nb][2 * r] * sl2 - mb);
        const float p1 = exp2f(s[nb][2 * r + 1] * sl2 - mb);
        s[nb][2 * r] = p0;
        s[nb][2 * r + 1] = p1;
        l_run[r] += p0 + p1;
      }
    }
    // O += P V
#pragma unroll
    for (int j = 0; j < BN / 16; ++j) {
      uint32_t a[4];
      a[0] = pack2(s[2 * j][0], s[2 * j][1]);
      a[1] = pack2(s[2 * j][2], s[2 * j][3]);
      a[2] = pack2(s[2 * j + 1][0], s[2 * j + 1][1]);
      a[3] = pack2(s[2 * j + 1][2], s[2 * j + 1][3]);
#pragma unroll
      for (int p = 0; p < HD / 16; ++p) {
        uint32_t b[4];
        const int mi = lane / 8, ri = lane % 8;
        ldsm_x4_t(b, smem_addr(tV + swz<HD>(j * 16 + ri + (mi & 1) * 8, p * 16 + (mi >> 1) * 8)));
        mma16816(oacc[2 * p], a, b[0], b[1]);
        mma16816(oacc[2 * p + 1], a, b[2], b[3]);
      }
    }
  }
  // finalize
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
  }
  const float inv0 = 1.f / l_run[0], inv1 = 1.f / l_run[1];
  bf16* o0 = o + (long long)qrow0 * ldo + (long long)h * HD;
  bf16* o1 = o + (long long)qrow1 * ldo + (long long)h * HD;
#pragma unroll
  for (int dn = 0; dn < DN; ++dn) {
    const int c = dn * 8 + 2 * qd;
    *reinterpret_cast<uint32_t*>(o0 + c) = pack2(oacc[dn][0] * inv0, oacc[dn][1] * inv0);
    *reinterpret_cast<uint32_t*>(o1 + c) = pack2(oacc[dn][2] * inv1, oacc[dn][3] * inv1);
  }
  if (qd == 0) {
    lse[(long long)h * T + qrow0] = (m_run[0] * sl2 + log2f(l_run[0])) / LOG2E;
    lse[(long long)h * T + qrow1] = (m_run[1] * sl2 + log2f(l_run[1])) / LOG2E;
  }
}

// --------------------------------------------------------------- backward
// delta[h, t] = sum_d dO[t,h,d] * O[t,h,d]; one warp per (t, h).
template <int HD>
__global__ void attn_bwd_pre_kernel(const bf16* __restrict__ o, long long ldo,
                                    const bf16* __restrict__ dout, long long lddo,
                                    float* __restrict__ delta, int T, int nq) {
  const long long w = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (w >= (long long)T * nq) return;
  const int t = (int)(w / nq), h = (int)(w % nq);
  float acc = 0.f;
  for (int d = lane; d < HD; d += 32)
    acc += __bfloat162float(o[(long long)t * ldo + h * HD + d]) *
           __bfloat162float(dout[(long long)t * lddo + h * HD + d]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) delta[(long long)h * T + t] = acc;
}

template <int HD>
__global__ void __launch_bounds__(256)
    attn_bwd_kernel(const bf16* __restrict__ q, long long ldq, const bf16* __restrict__ k,
                    long long ldk, const bf16* __restrict__ v, long long ldv,
                    const bf16* __restrict__ dout, long long lddo, const float* __restrict__ lse,
                    const float* __restrict__ delta, float* __restrict__ dq_acc,
                    bf16* __restrict__ dk, long long lddk, bf16* __restrict__ dv, long long lddv,
                    int T, int seq, int nq, int nk, float scale) {
  constexpr int BN = 128, BQ = 64, THREADS = 256, DK = HD / 16, DN = HD / 8;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  bf16* sK = reinterpret_cast<bf16*>(smem_raw);   // [BN][HD]
  bf16* sV = sK + BN * HD;                         // [BN][HD]
  bf16* sQ = sV + BN * HD;                         // [2][BQ][HD]
  bf16* sO = sQ + 2 * BQ * HD;                     // [2][BQ][HD]  (dO)
  bf16* sS = sO + 2 * BQ * HD;                     // [BN][BQ] dS^T
  float* sL = reinterpret_cast<float*>(sS + BN * BQ);  // [2][BQ] lse*log2e
  float* sD = sL + 2 * BQ;                              // [2][BQ] delta

  const int kb = blockIdx.x, kvh = blockIdx.y;
  const int k0 = kb * BN;
  const int s0 = (k0 / seq) * seq, s_end = s0 + seq;
  const int G = nq / nk;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = lane / 4, qd = lane % 4, mi = lane / 8, ri = lane % 8;
  const int first_qb = k0 / BQ;        // causal: queries >= keys
  const int nqb = (s_end - first_qb * BQ) / BQ;
  const int iters = G * nqb;
  const float sl2 = scale * LOG2E;

  load_tile<BN, HD, THREADS>(sK, k + (long long)k0 * ldk + (long long)kvh * HD, ldk);
  load_tile<BN, HD, THREADS>(sV, v + (long long)k0 * ldv + (long long)kvh * HD, ldv);
  auto issue = [&](int it, int buf) {
    const int hq = kvh * G + it / nqb;
    const int qs = (first_qb + it % nqb) * BQ;
    load_tile<BQ, HD, THREADS>(sQ + buf * BQ * HD, q + (long long)qs * ldq + (long long)hq * HD, ldq);
    load_tile<BQ, HD, THREADS>(sO + buf * BQ * HD, dout + (long long)qs * lddo + (long long)hq * HD,
                               lddo);
    for (int i = threadIdx.x; i < BQ; i += THREADS) {
      sL[buf * BQ + i] = lse[(long long)hq * T + qs + i] * LOG2E;
      sD[buf * BQ + i] = delta[(long long)hq * T + qs + i];
    }
  };
  issue(0, 0);
  cp_commit();

  float dkacc[DN][4], dvacc[DN][4];
#pragma unroll
  for (int i = 0; i < DN; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) dkacc[i][j] = dvacc[i][j] = 0.f;
  const int kw0 = warp * 16;               // this warp's keys within the tile
  const int key0 = k0 + kw0 + g, key1 = key0 + 8;

  for (int it = 0; it < iters; ++it) {
    const int buf = it & 1;
    cp_wait<0>();
    __syncthreads();
    if (it + 1 < iters) {
      issue(it + 1, buf ^ 1);
      cp_commit();
    }
    const int hq = kvh * G + it / nqb;
    const int qs = (first_qb + it % nqb) * BQ;
    const bf16* tQ = sQ + buf * BQ * HD;
    const bf16* tO = sO + buf * BQ * HD;
    const float* tL = sL + buf * BQ;
    const float* tD = sD + buf * BQ;

    // S^T (16 keys x 64 queries) and dP^T = V dO^T
    float st[BQ / 8][4], dpt[BQ / 8][4];
#pragma unroll
    for (int i = 0; i < BQ / 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) st[i][j] = dpt[i][j] = 0.f;
#pragma unroll
    for (int ks = 0; ks < DK; ++ks) {
      uint32_t ka[4], va[4];
      ldsm_x4(ka, smem_addr(sK + swz<HD>(kw0 + ri + (mi & 1) * 8, ks * 16 + (mi >> 1) * 8)));
      ldsm_x4(va, smem_addr(sV + swz<HD>(kw0 + ri + (mi & 1) * 8, ks * 16 + (mi >> 1) * 8)));
#pragma unroll
      for (int p = 0; p < BQ / 16; ++p) {
        uint32_t b[4];
        ldsm_x4(b, smem_addr(tQ + swz<HD>(p * 16 + ri + (mi >> 1) * 8, ks * 16 + (mi & 1) * 8)));
        mma16816(st[2 * p], ka, b[0], b[1]);
        mma16816(st[2 * p + 1], ka, b[2], b[3]);
        ldsm_x4(b, smem_addr(tO + swz<HD>(p * 16 + ri + (mi >> 1) * 8, ks * 16 + (mi & 1) * 8)));
        mma16816(dpt[2 * p], va, b[0], b[1]);
        mma16816(dpt[2 * p + 1], va, b[2], b[3]);
      }
    }
    // P^T and dS^T (causal: query >= key)
#pragma unroll
    for (int nb = 0; nb < BQ / 8; ++nb) {
      const int qc = qs + nb * 8 + 2 * qd;
      const float l0 = tL[nb * 8 + 2 * qd], l1 = tL[nb * 8 + 2 * qd + 1];
      const float d0 = tD[nb * 8 + 2 * qd], d1 = tD[nb * 8 + 2 * qd + 1];
      float p[4];
      p[0] = qc >= key0 ? exp2f(st[nb][0] * sl2 - l0) : 0.f;
      p[1] = qc + 1 >= key0 ? exp2f(st[nb][1] * sl2 - l1) : 0.f;
      p[2] = qc >= key1 ? exp2f(st[nb][2] * sl2 - l0) : 0.f;
      p[3] = qc + 1 >= key1 ? exp2f(st[nb][3] * sl2 - l1) : 0.f;
      st[nb][0] = p[0];
      st[nb][1] = p[1];
      st[nb][2] = p[2];
      st[nb][3] = p[3];
      dpt[nb][0] = p[0] * (dpt[nb][0] - d0);
      dpt[nb][1] = p[1] * (dpt[nb][1] - d1);
      dpt[nb][2] = p[2] * (dpt[nb][2] - d0);
      dpt[nb][3] = p[3] * (dpt[nb][3] - d1);
    }
    // dV += P^T dO ; dK += dS^T Q   (k dimension = queries)
#pragma unroll
    for (int j = 0; j < BQ / 16; ++j) {
      uint32_t pa[4], sa[4];
      pa[0] = pack2(st[2 * j][0], st[2 * j][1]);
      pa[1] = pack2(st[2 * j][2], st[2 * j][3]);
      pa[2] = pack2(st[2 * j + 1][0], st[2 * j + 1][1]);
      pa[3] = pack2(st[2 * j + 1][2], st[2 * j + 1][3]);
      sa[0] = pack2(dpt[2 * j][0], dpt[2 * j][1]);
      sa[1] = pack2(dpt[2 * j][2], dpt[2 * j][3]);
      sa[2] = pack2(dpt[2 * j + 1][0], dpt[2 * j + 1][1]);
      sa[3] = pack2(dpt[2 * j + 1][2], dpt[2 * j + 1][3]);
#pragma unroll
      for (int p = 0; p < HD / 16; ++p) {
        uint32_t b[4];
        ldsm_x4_t(b, smem_addr(tO + swz<HD>(j * 16 + ri + (mi & 1) * 8, p * 16 + (mi >> 1) * 8)));
        mma16816(dvacc[2 * p], pa, b[0], b[1]);
        mma16816(dvacc[2 * p + 1], pa, b[2], b[3]);
        ldsm_x4_t(b, smem_addr(tQ + swz<HD>(j * 16 + ri + (mi & 1) * 8, p * 16 + (mi >> 1) * 8)));
        mma16816(dkacc[2 * p], sa, b[0], b[1]);
        mma16816(dkacc[2 * p + 1], sa, b[2], b[3]);
      }
    }
    // stash dS^T (bf16) for the dQ product
#pragma unroll
    for (int nb = 0; nb < BQ / 8; ++nb) {
      const int c = nb * 8 + 2 * qd;
      const int r0 = kw0 + g, r1 = r0 + 8;
      *reinterpret_cast<uint32_t*>(sS + swz<BQ>(r0, nb * 8) + 2 * qd) = pack2(dpt[nb][0], dpt[nb][1]);
      *reinterpret_cast<uint32_t*>(sS + swz<BQ>(r1, nb * 8) + 2 * qd) = pack2(dpt[nb][2], dpt[nb][3]);
      (void)c;
    }
    __syncthreads();
    // dQ[qs + 16(w%4) .., half w/4 of HD] += scale * dS (16 q x BN keys) . K (BN keys x HD/2)
    const int qw0 = (warp & 3) * 16, half = warp >> 2;
    uint32_t da[BN / 16][4];
#pragma unroll
    for (int j = 0; j < BN / 16; ++j)  // A = dS rows=queries, k=keys, stored [key][query]
      ldsm_x4_t(da[j], smem_addr(sS + swz<BQ>(j * 16 + ri + (mi >> 1) * 8, qw0 + (mi & 1) * 8)));
    float acc[DN / 2][4];
#pragma unroll
    for (int i = 0; i < DN / 2; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
#pragma unroll
    for (int j = 0; j < BN / 16; ++j) {
#pragma unroll
      for (int p = 0; p < HD / 32; ++p) {
        uint32_t b[4];
        const int col = half * (HD / 2) + p * 16;
        ldsm_x4_t(b, smem_addr(sK + swz<HD>(j * 16 + ri + (mi & 1) * 8, col + (mi >> 1) * 8)));
        mma16816(acc[2 * p], da[j], b[0], b[1]);
        mma16816(acc[2 * p + 1], da[j], b[2], b[3]);
      }
    }
    // vector reduction: lane pairs (q, q^1) swap halves so each lane owns 4
    // consecutive columns of one row -> one 16-byte red.global.add per block
    const bool odd = qd & 1;
    float* dqrow = dq_acc + ((long long)(qs + qw0 + g + (odd ? 8 : 0)) * nq + hq) * HD;
#pragma unroll
    for (int i = 0; i < DN / 2; ++i) {
      const float s0v = odd ? acc[i][0] : acc[i][2];
      const float s1v = odd ? acc[i][1] : acc[i][3];
      const float r0 = __shfl_xor_sync(0xffffffffu, s0v, 1);
      const float r1 = __shfl_xor_sync(0xffffffffu, s1v, 1);
      float4 vv = odd ? make_float4(r0, r1, acc[i][2], acc[i][3])
                      : make_float4(acc[i][0], acc[i][1], r0, r1);
      vv.x *= scale; vv.y *= scale; vv.z *= scale; vv.w *= scale;
      const int c = half * (HD / 2) + i * 8 + 2 * (qd & ~1);
      atomicAdd(reinterpret_cast<float4*>(dqrow + c), vv);
    }
  }
  // write dK (scaled) and dV for this warp's 16 keys
  bf16* dk0 = dk + (long long)key0 * lddk + (long long)kvh * HD;
  bf16* dk1 = dk + (long long)key1 * lddk + (long long)kvh * HD;
  bf16* dv0 = dv + (long long)key0 * lddv + (long long)kvh * HD;
  bf16* dv1 = dv + (long long)key1 * lddv + (long long)kvh * HD;
#pragma unroll
  for (int dn = 0; dn < DN; ++dn) {
    const int c = dn * 8 + 2 * qd;
    *reinterpret_cast<uint32_t*>(dk0 + c) = pack2(dkacc[dn][0] * scale, dkacc[dn][1] * scale);
    *reinterpret_cast<uint32_t*>(dk1 + c) = pack2(dkacc[dn][2] * scale, dkacc[dn][3] * scale);
    *reinterpret_cast<uint32_t*>(dv0 + c) = pack2(dvacc[dn][0], dvacc[dn][1]);
    *reinterpret_cast<uint32_t*>(dv1 + c) = pack2(dvacc[dn][2], dvacc[dn][3]);
  }
}

// dq[t, h, :] = bf16(dq_acc[t, h, :])
__global__ void dq_cast_kernel(const float* __restrict__ acc, bf16* __restrict__ dq,
                               long long lddq, int T, int nq, int hd) {
  const long long n = (long long)T * nq * hd;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / ((long long)nq * hd), r = i % ((long long)nq * hd);
    dq[t * lddq + r] = __float2bfloat16_rn(acc[i]);
  }
}

}  // namespace
}  // namespace rp

using namespace rp;
#define RP_API extern "C" __attribute__((visibility("default")))

namespace {
template <int HD>
int attn_fwd_impl(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                  int64_t ldv, void* o, int64_t ldo, float* lse, int T, int seq, int nq, int nk,
                  float scale, cudaStream_t s) {
  constexpr int BM = 128, BN = 64;
  const int smem = (BM * HD + 4 * BN * HD) * 2;
  auto kern = attn_fwd_kernel<HD>;
  static bool cfg = false;
  if (!cfg) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return RP_E_CUDA;
    cfg = true;
  }
  dim3 grid(T / BM, nq);
  kern<<<grid, 256, smem, s>>>((const bf16*)q, ldq, (const bf16*)k, ldk, (const bf16*)v, ldv,
                               (bf16*)o, ldo, lse, T, seq, nq, nk, scale);
  return cudaGetLastError() == cudaSuccess ? RP_OK : RP_E_CUDA;
}

template <int HD>
int attn_bwd_impl(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                  int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                  const float* lse, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                  int64_t lddv, float* dq_acc, float* delta, int T, int seq, int nq, int nk,
                  float scale, cudaStream_t s) {
  constexpr int BN = 128, BQ = 64;
  if (cudaMemsetAsync(dq_acc, 0, sizeof(float) * (size_t)T * nq * HD, s) != cudaSuccess)
    return RP_E_CUDA;
  const long long warps = (long long)T * nq;
  attn_bwd_pre_kernel<HD><<<(int)((warps + 7) / 8), 256, 0, s>>>(
      (const bf16*)o, ldo, (const bf16*)dout, lddo, delta, T, nq);
  const int smem = (2 * BN * HD + 4 * BQ * HD + BN * BQ) * 2 + 4 * BQ * 4;
  auto kern = attn_bwd_kernel<HD>;
  static bool cfg = false;
  if (!cfg) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
        cudaSuccess)
      return RP_E_CUDA;
    cfg = true;
  }
  dim3 grid(T / BN, nk);
  kern<<<grid, 256, smem, s>>>((const bf16*)q, ldq, (const bf16*)k, ldk, (const bf16*)v, ldv,
                               (const bf16*)dout, lddo, lse, delta, dq_acc, (bf16*)dk, lddk,
                               (bf16*)dv, lddv, T, seq, nq, nk, scale);
  const long long n = (long long)T * nq * HD;
  dq_cast_kernel<<<(int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16), 256, 0, s>>>(
      dq_acc, (bf16*)dq, lddq, T, nq, HD);
  return cudaGetLastError() == cudaSuccess ? RP_OK : RP_E_CUDA;
}

bool attn_args_ok(int T, int seq, int nq, int nk, int hd) {
  return T > 0 && seq > 0 && seq % 128 == 0 && T % seq == 0 && nk > 0 && nq % nk == 0 &&
         (hd == 64 || hd == 128);
}
}  // namespace

RP_API int rp_attn_fwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                       int64_t ldv, void* o, int64_t ldo, float* lse, int32_t T, int32_t seq,
                       int32_t nq, int32_t nk, int32_t head_dim, float scale, void* stream) {
  if (!attn_args_ok(T, seq, nq, nk, head_dim)) return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  return head_dim == 128
             ? attn_fwd_impl<128>(q, ldq, k, ldk, v, ldv, o, ldo, lse, T, seq, nq, nk, scale, s)
             : attn_fwd_impl<64>(q, ldq, k, ldk, v, ldv, o, ldo, lse, T, seq, nq, nk, scale, s);
}

RP_API int rp_attn_bwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                       int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                       const float* lse, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                       int64_t lddv, float* dq_acc, float* delta, int32_t T, int32_t seq,
                       int32_t nq, int32_t nk, int32_t head_dim, float scale, void* stream) {
  if (!attn_args_ok(T, seq, nq, nk, head_dim)) return RP_E_INPUT;
  auto s = (cudaStream_t)stream;
  return head_dim == 128
             ? attn_bwd_impl<128>(q, ldq, k, ldk, v, ldv, o, ldo, dout, lddo, lse, dq, lddq, dk,
                                  lddk, dv, lddv, dq_acc, delta, T, seq, nq, nk, scale, s)
             : attn_bwd_impl<64>(q, ldq, k, ldk, v, ldv, o, ldo, dout, lddo, lse, dq, lddq, dk,
                                 lddk, dv, lddv, dq_acc, delta, T, seq, nq, nk, scale, s);
}
