// Curved-geometry (per-point metric) kernels.  See wk_abi.cu for dispatch.
#pragma once
#include "wk_common.cuh"

namespace wk {

struct CurvedArgs {
  const double* inv_jac;   // (E, d, d, n^d)  degree-k Gauss points
  const double* jxw;       // (E, n^d)
  const double* fnormal[6];
  const double* fjxw[6];
};

}  // namespace wk
