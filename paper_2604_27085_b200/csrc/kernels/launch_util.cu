// Host-side launch helpers (see launch_util.h).
#include "kernels/launch_util.h"

#include <map>
#include <mutex>
#include <set>
#include <tuple>

namespace rp {
namespace {
std::mutex g_mu;
std::set<std::tuple<const void*, int, int>> g_smem_done;  // (kernel, device, bytes)
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
  const auto key = std::make_tuple(kern, dev, bytes);
  if (g_smem_done.count(key)) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return false;
  g_smem_done.insert(key);
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
