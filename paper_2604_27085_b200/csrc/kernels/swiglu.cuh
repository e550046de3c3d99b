// SwiGLU backward of one element, shared by the standalone kernel
// (elementwise.cu) and the down-projection dgrad GEMM's fused epilogue
// (gemm_sm100.cu), so the two paths produce identical bits.
//   act = silu(g) * u,  d = dL/d act  ->  dg = d * u * s * (1 + g (1 - s)),
//   du = d * g * s,  s = sigmoid(g)
// The reciprocal is the MUFU approximation (2 ulp): an IEEE division is a
// ~20-instruction sequence that made the GEMM epilogue, not the tensor core,
// the fused kernel's bottleneck.
#pragma once
#include <cuda_runtime.h>

namespace rp {
__device__ __forceinline__ float swiglu_fwd_elem(float g, float u) {
  return g * __fdividef(1.f, 1.f + __expf(-g)) * u;
}
__device__ __forceinline__ void swiglu_bwd_elem(float d, float g, float u, float& dg, float& du) {
  const float s = __fdividef(1.f, 1.f + __expf(-g));
  du = d * g * s;
  dg = d * u * s * (1.f + g * (1.f - s));
}
}  // namespace rp
