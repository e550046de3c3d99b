// Host-side launch helpers (see launch_util.h).
#include "kernels/launch_util.h"

#include <map>
#include <mutex>
#include <set>
#include <tuple>

namespace rp {
namespace {
std::mutex g_mu;
// (kernel, device) -> the MaxDynamicSharedMemorySize set so far. The attribute
// is an upper bound for every later launch, so it only ever grows: setting it
// to a smaller size for one launch would make a later, larger launch of the
// same kernel fail with "invalid argument".
std::map<std::pair<const void*, int>, int> g_smem_max;
struct WsKey {
  cudaStream_t s;
  int dev, tag;
  bool operator<(const WsKey& o) const { return std::tie(s, dev, tag) < std::tie(o.s, o.dev, o.tag); }
};
std::map<WsKey, Workspace> g_ws;
}  // namespace

bool ensure_smem(const void* kern, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> g(g_mu);
  constexpr int kDefault = 48 * 1024;  // allowed without opting in
  int& cur = g_smem_max[std::make_pair(kern, dev)];
  if (bytes <= (cur > kDefault ? cur : kDefault)) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return false;
  cur = bytes;
  return true;
}

Workspace* stream_workspace(cudaStream_t s, int tag, std::size_t bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(g_mu);
  Workspace& w = g_ws[WsKey{s, dev, tag}];
  if (w.bytes < bytes) {
    // cudaFree synchronises the device: earlier launches that used the old
    // buffer are done before it is released
    if (w.p) cudaFree(w.p);
    w = Workspace{};
    void* p = nullptr;
    // zeroed ON s: the callers' streams are non-blocking, so a plain
    // cudaMemset (legacy stream) could land after s's next kernel had already
    // written the buffer (seen as a once-per-stream corruption of the
    // attention backward's -lse*log2e block)
    if (cudaMalloc(&p, bytes) != cudaSuccess || cudaMemsetAsync(p, 0, bytes, s) != cudaSuccess) {
      if (p) cudaFree(p);
      cudaGetLastError();
      return nullptr;
    }
    w.p = p;
    w.bytes = bytes;
  }
  return &w;
}

void release_stream_workspaces(cudaStream_t s) {
  std::lock_guard<std::mutex> g(g_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto it = g_ws.begin(); it != g_ws.end();) {
    if (it->first.s == s) {
      cudaSetDevice(it->first.dev);
      if (it->second.p) cudaFree(it->second.p);
      it = g_ws.erase(it);
    } else {
      ++it;
    }
  }
  cudaSetDevice(cur);
}

}  // namespace rp
