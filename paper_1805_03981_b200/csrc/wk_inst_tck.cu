// General (non-Cartesian / multi-class) affine ADER kernel A launchers (the
// Taylor loop; ADER-HDG composes it with the stage kernel, wk_abi.cu), one
// (WK_D, WK_N) pair per object.
#include <algorithm>
#include <cstdlib>

#include "wk_launch.h"

#ifndef WK_D
#error "compile with -DWK_D=<2|3> -DWK_N=<2..9>"
#endif

namespace wk {

namespace {

template <int D, int N, bool CART>
void launch_ader_a(const TckArgs& a, cudaStream_t s) {
  using S = Shape<D, N>;
  const size_t smem = TckSmem<D, N, CART>::bytes(a.acc_len, a.tab_len);
  require(smem <= 227 * 1024, "TCK working set exceeds shared memory");
  ensure_smem(ader_a_kernel<D, N, CART>, smem);
  const long long blocks = (a.op.E + S::EPB - 1) / S::EPB;
  if (blocks == 0) return;
  ader_a_kernel<D, N, CART><<<(unsigned)blocks, S::TPB, smem, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), "ader_a_kernel");
}

}  // namespace

template <int D, int N>
void affine_ader_a_general_launch(bool cart, bool hdg, const TckArgs& a, cudaStream_t s) {
  require(!hdg, "general affine ADER-HDG is composed on the host (run_ader_a)");
  if (cart) return launch_ader_a<D, N, true>(a, s);
  return launch_ader_a<D, N, false>(a, s);
}

template void affine_ader_a_general_launch<WK_D, WK_N>(bool, bool, const TckArgs&, cudaStream_t);

}  // namespace wk
