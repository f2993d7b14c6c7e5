// Per-(d, n) kernel launchers; defined and explicitly instantiated in
// wk_inst.cu, compiled once per (WK_D, WK_N) so the build parallelises.
#pragma once
#include "wk_curved.cuh"
#include "wk_error.h"
#include "wk_tck.cuh"
#include "wk_stream_ader.cuh"
#include "wk_stream_curved.cuh"
#include "wk_small.cuh"

namespace wk {

template <int D, int N>
void affine_op_launch(bool cart, int mode, const AffineArgs& a, cudaStream_t s);
template <int D, int N>
void affine_ader_a_launch(bool cart, bool hdg, const TckArgs& a, cudaStream_t s);
template <int D, int N>
void affine_ader_a_general_launch(bool cart, bool hdg, const TckArgs& a, cudaStream_t s);
template <int D, int N>
bool affine_stream_ader_launch(bool hdg, int stride, bool shift, const TckStreamArgs& a,
                               cudaStream_t s);
template <int D, int N>
bool curved_stream_launch(int kind, int stride, bool shift, const CurvedStreamArgs& a,
                          cudaStream_t s);
template <int D, int N>
void curved_op_launch(int mode, const AffineArgs& a, const CurvedArgs& g, cudaStream_t s);
template <int D, int N>
void curved_ader_a_launch(bool hdg, const TckArgs& a, const CurvedArgs& g, cudaStream_t s);
// whole-run LSRK on one thread-block cluster (wk_small.cuh); returns false
// if the mesh does not fit the cluster's shared memory
template <int D, int N>
bool small_lsrk_launch(const SmallArgs& a, cudaStream_t s, bool dry_run);

#define WK_FOR_EACH_DN(X) \
  X(2, 2) X(2, 3) X(2, 4) X(2, 5) X(2, 6) X(2, 7) X(2, 8) X(2, 9) \
  X(3, 2) X(3, 3) X(3, 4) X(3, 5) X(3, 6) X(3, 7) X(3, 8) X(3, 9)

#define WK_DECLARE_EXTERN(d, n)                                                           \
  extern template void affine_op_launch<d, n>(bool, int, const AffineArgs&, cudaStream_t); \
  extern template void affine_ader_a_launch<d, n>(bool, bool, const TckArgs&, cudaStream_t); \
  extern template void affine_ader_a_general_launch<d, n>(bool, bool, const TckArgs&,      \
                                                          cudaStream_t);                   \
  extern template bool affine_stream_ader_launch<d, n>(bool, int, bool, const TckStreamArgs&, \
                                                      cudaStream_t);                       \
  extern template bool curved_stream_launch<d, n>(int, int, bool, const CurvedStreamArgs&,    \
                                                 cudaStream_t);                            \
  extern template void curved_op_launch<d, n>(int, const AffineArgs&, const CurvedArgs&,   \
                                              cudaStream_t);                               \
  extern template void curved_ader_a_launch<d, n>(bool, const TckArgs&, const CurvedArgs&, \
                                                  cudaStream_t);                           \
  extern template bool small_lsrk_launch<d, n>(const SmallArgs&, cudaStream_t, bool);
WK_FOR_EACH_DN(WK_DECLARE_EXTERN)
#undef WK_DECLARE_EXTERN

}  // namespace wk
