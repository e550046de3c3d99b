// Host-side launch helpers shared by the kernel translation units.
//
// * ensure_smem: cudaFuncAttributeMaxDynamicSharedMemorySize is a per-DEVICE
//   attribute of a kernel, so it is set once per (kernel, device) — a
//   process-wide "configured" flag would leave the second GPU of a
//   multi-device runtime at the 48 KB default and every launch there fails.
// * stream_workspace: scratch owned by a stream (split-K partials, the fused
//   attention backward's fp32 dQ^T accumulator). GEMMs / attention on two
//   streams may run concurrently, so scratch is per stream; it is keyed by
//   (stream, device) and released with release_stream_workspaces() when the
//   runtime destroys the stream.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace rp {

bool ensure_smem(const void* kern, int bytes);
template <class K>
bool ensure_smem_t(K* kern, int bytes) {
  return ensure_smem(reinterpret_cast<const void*>(kern), bytes);
}

struct Workspace {
  void* p = nullptr;
  std::size_t bytes = 0;
  unsigned epoch = 0;  // bumped by users whose flags carry a launch epoch
};
// Workspace `tag` of stream s on the current device, grown to >= bytes
// (zero-filled when (re)allocated); nullptr if the allocation fails.
Workspace* stream_workspace(cudaStream_t s, int tag, std::size_t bytes);
// Frees every workspace of stream s (call before cudaStreamDestroy).
void release_stream_workspaces(cudaStream_t s);

enum WorkspaceTag { WS_SPLITK_PARTIALS = 0, WS_SPLITK_FLAGS = 1, WS_ATTN_DQ = 2 };

}  // namespace rp
