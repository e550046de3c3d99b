// Host-mapped flag words of the optimizer hand-off protocol (PAPER.md:468-476,
// north_star "per-layer cudaEvents plus host-mapped flag words").
//
// One 32-bit word per parameter group ("latest published version") and per
// worker ("latest iteration whose loss is on the host"), in pinned host
// memory mapped into every device's address space. A GPU stream SETS a word
// with cuStreamWriteValue32 when the action completes and a stream WAITS on
// it with cuStreamWaitValue32(>=), so the wait names a version, not an event
// object of a particular device: an upload on any GPU waits "group g
// published >= t". The controller reads the same words without entering the
// driver (early-return loss, publication progress) instead of blocking in
// cudaEventSynchronize. Every wait is enqueued after the write it waits for
// (the controller enqueues in a topological order), so a wait can never
// stall a hardware queue that the write sits behind.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace rp {
namespace rt {

class FlagWords {
 public:
  void init(int n);  // n words, zeroed; needs a current device
  ~FlagWords();
  // GPU side (enqueued on `st`)
  void set(cudaStream_t st, int i, uint32_t value) const;
  void wait_geq(cudaStream_t st, int i, uint32_t value) const;
  // host side
  uint32_t read(int i) const { return __atomic_load_n(host_ + i, __ATOMIC_ACQUIRE); }
  void host_set(int i, uint32_t v) { __atomic_store_n(host_ + i, v, __ATOMIC_RELEASE); }
  int size() const { return n_; }

 private:
  uint32_t* host_ = nullptr;
  CUdeviceptr dev_ = 0;  // unified address: the same on every device
  int n_ = 0;
};

}  // namespace rt
}  // namespace rp
