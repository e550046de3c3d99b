// Host-mapped flag words (see flags.h).
#include "runtime/flags.h"

#include <cstring>
#include <string>

#include "runtime/runtime_internal.h"

namespace rp {
namespace rt {
namespace {
using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
template <class F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    throw RtError(RP_E_CUDA, std::string("driver entry point missing: ") + name);
  return reinterpret_cast<F>(p);
}
WriteFn write_fn() {
  static WriteFn f = entry<WriteFn>("cuStreamWriteValue32");
  return f;
}
WaitFn wait_fn() {
  static WaitFn f = entry<WaitFn>("cuStreamWaitValue32");
  return f;
}
}  // namespace

void FlagWords::init(int n) {
  n_ = n;
  RP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host_), sizeof(uint32_t) * (size_t)n,
                        cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(host_, 0, sizeof(uint32_t) * (size_t)n);
  void* d = nullptr;
  RP_CUDA(cudaHostGetDevicePointer(&d, host_, 0));
  dev_ = reinterpret_cast<CUdeviceptr>(d);
  write_fn();  // resolve the entry points now: fail at creation, not mid-step
  wait_fn();
}

FlagWords::~FlagWords() {
  if (host_) cudaFreeHost(host_);
}

// CU_STREAM_WRITE_VALUE_DEFAULT: the write is preceded by a system-wide
// memory fence, so e.g. a loss copied to the host before the flag is set is
// visible once the flag is
void FlagWords::set(cudaStream_t st, int i, uint32_t value) const {
  if (write_fn()(reinterpret_cast<CUstream>(st), dev_ + sizeof(uint32_t) * (size_t)i, value,
                 CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    throw RtError(RP_E_CUDA, "cuStreamWriteValue32 failed");
}

void FlagWords::wait_geq(cudaStream_t st, int i, uint32_t value) const {
  if (wait_fn()(reinterpret_cast<CUstream>(st), dev_ + sizeof(uint32_t) * (size_t)i, value,
                CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    throw RtError(RP_E_CUDA, "cuStreamWaitValue32 failed");
}

}  // namespace rt
}  // namespace rp
