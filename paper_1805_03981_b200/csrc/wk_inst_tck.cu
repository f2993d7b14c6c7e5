// General (non-Cartesian / multi-class) affine ADER kernel A launchers, one
// (WK_D, WK_N) pair per object.  Compiled with -Xptxas -O1: at -O3 the sm_100a
// code of ader_a_kernel's fused face stage faulted on meshes above ~2k
// elements (investigation in DESIGN.md); the Cartesian hot path uses
// affine_group_ader_kernel (wk_group_ader.cuh) instead.
#include <algorithm>
#include <cstdlib>

#include "wk_launch.h"

#ifndef WK_D
#error "compile with -DWK_D=<2|3> -DWK_N=<2..9>"
#endif

namespace wk {

namespace {

template <int D, int N, bool CART, bool HDG>
void launch_ader_a(const TckArgs& a, cudaStream_t s) {
  using S = Shape<D, N>;
  size_t smem = TckSmem<D, N, CART>::bytes(a.acc_len, a.tab_len);
  if (const char* pad = getenv("WK_DBG_SMEM_PAD")) smem += (size_t)atoi(pad);
  require(smem <= 227 * 1024, "TCK working set exceeds shared memory");
  ensure_smem(ader_a_kernel<D, N, CART, HDG>, smem);
  const long long blocks = (a.op.E + S::EPB - 1) / S::EPB;
  if (blocks == 0) return;
  ader_a_kernel<D, N, CART, HDG><<<(unsigned)blocks, S::TPB, smem, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), "ader_a_kernel");
}

}  // namespace

template <int D, int N>
void affine_ader_a_general_launch(bool cart, bool hdg, const TckArgs& a, cudaStream_t s) {
  if (cart) {
    if (hdg) return launch_ader_a<D, N, true, true>(a, s);
    return launch_ader_a<D, N, true, false>(a, s);
  }
  if (hdg) return launch_ader_a<D, N, false, true>(a, s);
  return launch_ader_a<D, N, false, false>(a, s);
}

template void affine_ader_a_general_launch<WK_D, WK_N>(bool, bool, const TckArgs&, cudaStream_t);

}  // namespace wk
