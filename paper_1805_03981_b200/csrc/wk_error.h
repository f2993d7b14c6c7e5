// Error plumbing shared by the ABI and the kernel-launch translation units.
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/wavekernel_b200.h"

namespace wk {

struct WkError : std::runtime_error {
  int code;
  WkError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define WK_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      throw ::wk::WkError(WK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define WK_CUDA_AT(call, where)                                                        \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      throw ::wk::WkError(WK_ECUDA, std::string(where) + ": " + cudaGetErrorString(_e)); \
  } while (0)

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw WkError(WK_EINVAL, msg);
}

int num_sms();

// Per-(device, kernel) launch setup: the dynamic shared-memory attribute
// last set and the resident CTAs per SM it gives.  cudaFuncSetAttribute is
// per device, so a process that drives several devices keeps one entry each
// (the cache used to be a function-local static shared by all devices).
struct KernelSetup {
  size_t smem = 0;
  int per_sm = 0;
  bool nonportable_cluster = false;
};
KernelSetup& kernel_setup(const void* kernel);

// Set the kernel's dynamic-smem limit to at least `smem` on the current
// device (once per device and size).
template <typename Kern>
KernelSetup& ensure_smem(Kern kernel, size_t smem) {
  KernelSetup& k = kernel_setup(reinterpret_cast<const void*>(kernel));
  if (k.smem < smem) {
    WK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k.smem = smem;
  }
  return k;
}

// ensure_smem + the occupancy at that size (persistent-grid sizing).
template <typename Kern>
int resident_per_sm(Kern kernel, int threads, size_t smem) {
  KernelSetup& k = ensure_smem(kernel, smem);
  if (!k.per_sm) {
    WK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k.per_sm, kernel, threads, smem));
    require(k.per_sm > 0, "kernel does not fit on an SM");
  }
  return k.per_sm;
}

// thread-local message returned by wk_last_error() (wk_abi.cu)
void set_last_error(const char* msg);

// run fn, mapping exceptions to WK_E* codes + the last-error message
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return WK_OK;
  } catch (const WkError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return WK_EINVAL;
  }
}

}  // namespace wk
