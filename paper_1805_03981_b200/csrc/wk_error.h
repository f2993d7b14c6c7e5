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
