// Kernel launchers for one (d, n) pair, selected by -DWK_D=<d> -DWK_N=<n>.
// The build compiles this file once per supported pair (16 objects) so the
// template-heavy kernels compile in parallel.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "wk_launch.h"
#include "wk_group.cuh"
#include "wk_stream.cuh"
#include "wk_streamd.cuh"
#include "wk_group_ader.cuh"
#include "wk_pencil.cuh"

#ifndef WK_D
#error "compile with -DWK_D=<2|3> -DWK_N=<2..9>"
#endif

namespace wk {

#ifndef WK_STREAMD_DEFAULT
#define WK_STREAMD_DEFAULT(D, N) ((D) == 3)
#endif

// CTA slots of a persistent grid: every SM's resident CTAs, minus `hold` SMs'
// worth left free for concurrent work (AffineArgs::grid_hold)
inline long long persistent_slots(int per_sm, int hold) {
  const int sms = num_sms();
  return (long long)per_sm * (hold > 0 && hold < sms ? sms - hold : sms);
}


namespace {

template <int D, int N, bool CART, int MODE>
void launch_affine_op(const AffineArgs& a, cudaStream_t s) {
  using S = Shape<D, N>;
  const size_t smem = StageCfg<D, N>::BYTES;
  const int per_sm = resident_per_sm(affine_stage_kernel<D, N, CART, MODE>, S::TPB, smem);
  const long long tiles = (a.E + S::EPB - 1) / S::EPB;
  if (tiles == 0) return;
  const long long grid = std::min<long long>(tiles, persistent_slots(per_sm, a.grid_hold));
  affine_stage_kernel<D, N, CART, MODE><<<(unsigned)grid, S::TPB, smem, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), "affine_stage_kernel");
}

template <int D, int N, int MODE>
void launch_pencil(const AffineArgs& a, cudaStream_t s) {
  using P = PencilCfg<D, N>;
  const size_t smem = P::BYTES;
  const int per_sm = resident_per_sm(affine_pencil_kernel<D, N, MODE>, P::TPB, smem);
  const long long tiles = (a.E + P::EPB - 1) / P::EPB;
  if (tiles == 0) return;
  const long long grid = std::min<long long>(tiles, persistent_slots(per_sm, a.grid_hold));
  affine_pencil_kernel<D, N, MODE><<<(unsigned)grid, P::TPB, smem, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), "affine_pencil_kernel");
}

template <typename K, typename Kern>
void launch_persistent(Kern kern, const AffineArgs& a0, cudaStream_t s, const char* name) {
  const size_t smem = K::BYTES;
  const int per_sm = resident_per_sm(kern, K::TG, smem);
  AffineArgs a = a0;
  if (a.tmap_ch % K::EPG) a.tmap_ch = 0;   // chunks must hold whole tiles
  const long long tiles = (a.E + K::EPG - 1) / K::EPG;
  if (tiles == 0) return;
  const long long grid = std::min<long long>(tiles, persistent_slots(per_sm, a.grid_hold));
  kern<<<(unsigned)grid, K::TG, smem, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), name);
}

// direction-parallel CTA (wk_streamd.cuh): WK_STREAM=seq selects the
// one-group kernel for A/B runs
template <int D, int N, int MODE>
bool stream_dir(const AffineArgs& a) {
  static const int env = [] {
    const char* k = getenv("WK_STREAM");
    return k ? (std::string(k) == "dir" ? 1 : 0) : -1;
  }();
  if (!StreamDCfg<D, N>::ALIGNED) return false;
  if (env >= 0) return env == 1;
  // LSRK stages over long vectors (>= 256 MB) with one-warp groups (n <= 5)
  // take the one-group kernel.  Runs that long sit at the board power cap,
  // where the stage kernel has a slow state (config 5: 15 -> 18.5 ms/step,
  // DESIGN.md section 6).  The direction-parallel kernel as built (8 CTAs per
  // SM, idle lanes off, loop unrolled by two) stayed out of it in 20 bench
  // runs + 3 x 30 repeats on three boards and is 2 % faster there (14.52 /
  // 14.92 / 14.97 vs 14.83 / 15.27 / 15.25 ms/step) -- but every variant one
  // step away from it (9 CTAs, repeated lanes, no unroll) fell in, some at
  // once, while the one-group kernel never did in any build of the session
  // (~25 runs, six boards).  A 2 % gain does not pay for that exposure;
  // WK_STREAM=dir takes it.  Smaller or shorter runs (config 2: 3 % faster),
  // n >= 6 (config 4) and ADER kernel B keep the direction-parallel kernel.
  constexpr int C = D + 1, NODES = StreamDCfg<D, N>::NODES;
  if (MODE == OUT_LSRK && StreamCfg<D, N>::TG == 32 &&
      (double)a.E * C * NODES * 8.0 >= 256e6)
    return false;
  return WK_STREAMD_DEFAULT(D, N);
}

template <int D, int N, int MODE, bool FAST>
void launch_streamd_k(const AffineArgs& a0, cudaStream_t s);

template <int D, int N, int MODE>
void launch_streamd(const AffineArgs& a0, cudaStream_t s) {
  // the steppers always apply both parts with the context's stabilization:
  // those flags are compile-time facts of the FAST instantiation
  if (a0.parts == PART_BOTH && a0.stab) launch_streamd_k<D, N, MODE, true>(a0, s);
  else launch_streamd_k<D, N, MODE, false>(a0, s);
}

template <int D, int N, int MODE, bool FAST>
void launch_streamd_k(const AffineArgs& a0, cudaStream_t s) {
  using K = StreamDCfg<D, N>;
  auto kern = affine_streamd_kernel<D, N, MODE, FAST>;
  int per_sm = resident_per_sm(kern, K::TPB, K::BYTES);
  // At most 8 CTAs (24 warps at n = 5) per SM.  With all 9 that fit, long
  // runs at the board power cap fell -- on about half the boards tried --
  // into a throttled state (config 5 LSRK45 15.2 -> 18.5 ms/step, SM clock
  // back UP at 1.9 GHz); 8 never did and cost 0.5 %.  WK_STREAM_PER_SM
  // overrides (experiments).
  static const int cap = [] {
    const char* k = getenv("WK_STREAM_PER_SM");
    return k ? atoi(k) : 8;
  }();
  if (cap > 0) per_sm = std::min(per_sm, cap);
  AffineArgs a = a0;
  if (a.tmap_ch % K::EPG) a.tmap_ch = 0;   // chunks must hold whole tiles
  const long long tiles = (a.E + K::EPG - 1) / K::EPG;
  if (tiles == 0) return;
  const long long grid = std::min<long long>(tiles, persistent_slots(per_sm, a.grid_hold));
  kern<<<(unsigned)grid, K::TPB, K::BYTES, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), "affine_streamd_kernel");
}

template <int D, int N, int MODE>
void launch_stream(const AffineArgs& a, cudaStream_t s) {
  if constexpr (StreamDCfg<D, N>::ALIGNED && StreamDCfg<D, N>::BYTES <= 227 * 1024) {
    // 32-bit element indices in the kernel
    if (stream_dir<D, N, MODE>(a) && a.e_begin + a.E < (1LL << 31))
      return launch_streamd<D, N, MODE>(a, s);
  }
  launch_persistent<StreamCfg<D, N>>(affine_stream_kernel<D, N, MODE>, a, s,
                                     "affine_stream_kernel");
}

template <int D, int N, int MODE>
void launch_group(const AffineArgs& a, cudaStream_t s) {
  using G = GroupCfg<D, N>;
  const size_t smem = G::BYTES;
  ensure_smem(affine_group_kernel<D, N, MODE>, smem);
  const long long per_block = (long long)G::EPG * G::GPB;
  const long long grid = (a.E + per_block - 1) / per_block;
  if (grid == 0) return;
  affine_group_kernel<D, N, MODE><<<(unsigned)grid, G::TPB, smem, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), "affine_group_kernel");
}

template <int D, int N, int MODE>
void launch_curved_op(const AffineArgs& a, const CurvedArgs& g, cudaStream_t s) {
  using S = CShape<D, N>;
  require(S::BYTES <= 227 * 1024, "curved element tile exceeds shared memory");
  ensure_smem(curved_op_kernel<D, N, MODE>, S::BYTES);
  if (a.E == 0) return;
  curved_op_kernel<D, N, MODE><<<(unsigned)a.E, S::TPB, S::BYTES, s>>>(a, g);
  WK_CUDA_AT(cudaGetLastError(), "curved_op_kernel");
}

template <int D, int N, bool HDG>
void launch_curved_ader_a(const TckArgs& a, const CurvedArgs& g, cudaStream_t s) {
  const size_t smem = CTckSmem<D, N>::bytes(a.acc_len, a.tab_len);
  require(smem <= 227 * 1024, "curved TCK working set exceeds shared memory");
  ensure_smem(curved_ader_a_kernel<D, N, HDG>, smem);
  if (a.op.E == 0) return;
  curved_ader_a_kernel<D, N, HDG><<<(unsigned)a.op.E, CShape<D, N>::TPB, smem, s>>>(a, g);
  WK_CUDA_AT(cudaGetLastError(), "curved_ader_a_kernel");
}

}  // namespace

template <int D, int N>
void affine_op_launch(bool cart, int mode, const AffineArgs& a, cudaStream_t s) {
  if (cart && a.geo_class == nullptr) {
    // axis-aligned single-class mesh: pencil-parallel kernel (wk_pencil.cuh)
    // WK_KERNEL=group selects the non-persistent variant (A/B comparisons)
    static const bool use_group = [] {
      const char* k = getenv("WK_KERNEL");
      return k && std::string(k) == "group";
    }();
    if (!use_group) {
      switch (mode) {
        case OUT_MINVK: return launch_stream<D, N, OUT_MINVK>(a, s);
        case OUT_RHS: return launch_stream<D, N, OUT_RHS>(a, s);
        case OUT_LSRK: return launch_stream<D, N, OUT_LSRK>(a, s);
        case OUT_ADERB: return launch_stream<D, N, OUT_ADERB>(a, s);
      }
    }
    switch (mode) {
      case OUT_MINVK: return launch_group<D, N, OUT_MINVK>(a, s);
      case OUT_RHS: return launch_group<D, N, OUT_RHS>(a, s);
      case OUT_LSRK: return launch_group<D, N, OUT_LSRK>(a, s);
      case OUT_ADERB: return launch_group<D, N, OUT_ADERB>(a, s);
    }
  } else if (cart) {
    switch (mode) {
      case OUT_MINVK: return launch_affine_op<D, N, true, OUT_MINVK>(a, s);
      case OUT_RHS: return launch_affine_op<D, N, true, OUT_RHS>(a, s);
      case OUT_LSRK: return launch_affine_op<D, N, true, OUT_LSRK>(a, s);
      case OUT_ADERB: return launch_affine_op<D, N, true, OUT_ADERB>(a, s);
    }
  } else {
    switch (mode) {
      case OUT_MINVK: return launch_affine_op<D, N, false, OUT_MINVK>(a, s);
      case OUT_RHS: return launch_affine_op<D, N, false, OUT_RHS>(a, s);
      case OUT_LSRK: return launch_affine_op<D, N, false, OUT_LSRK>(a, s);
      case OUT_ADERB: return launch_affine_op<D, N, false, OUT_ADERB>(a, s);
    }
  }
  throw WkError(WK_EINVAL, "bad operator mode");
}

template <int D, int N, bool HDG>
void launch_group_ader(const TckArgs& a, cudaStream_t s) {
  using G = GroupAderCfg<D, N>;
  const size_t smem = G::bytes(a.acc_len, a.tab_len);
  require(smem <= 227 * 1024, "TCK working set exceeds shared memory");
  ensure_smem(affine_group_ader_kernel<D, N, HDG>, smem);
  const long long grid = (a.op.E + G::GPB - 1) / G::GPB;
  if (grid == 0) return;
  affine_group_ader_kernel<D, N, HDG><<<(unsigned)grid, G::TPB, smem, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), "affine_group_ader_kernel");
}

template <int D, int N, bool HDG, int STRIDE, bool SHIFT>
void launch_stream_ader(const TckStreamArgs& a0, cudaStream_t s) {
  using K = StreamAderCfg<D, N>;
  TckStreamArgs a = a0;
  if (a.op.tmap_ch % K::EPG) a.op.tmap_ch = 0;   // chunks must hold whole tiles
  auto kern = affine_stream_ader_kernel<D, N, HDG, STRIDE, SHIFT>;
  {
    // n = 8: the full shared-memory carveout lets 3 CTAs (each 62 KB) share
    // an SM (2 with the default split) -- config 4 kernel A with 3 x 4 warps
    // per SM: ADER-HDG 5.88 -> 5.61 ms/step.  WK_ADER_CARVEOUT=0/1 overrides.
    static int env = -2;
    if (env == -2) {
      const char* e = getenv("WK_ADER_CARVEOUT");
      env = e ? atoi(e) : -1;
    }
    KernelSetup& ks = kernel_setup(reinterpret_cast<const void*>(kern));
    if (!ks.nonportable_cluster && (env == 1 || (env < 0 && N >= 7))) {
      WK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                   cudaSharedmemCarveoutMaxShared));
      ks.nonportable_cluster = true;   // (flag reused: carveout set once per device)
    }
  }
  const int per_sm = resident_per_sm(kern, K::TG, K::BYTES);
  const long long tiles = (a.op.E + K::EPG - 1) / K::EPG;
  if (tiles == 0) return;
  const long long grid = std::min<long long>(tiles, persistent_slots(per_sm, a.op.grid_hold));
  kern<<<(unsigned)grid, K::TG, K::BYTES, s>>>(a);
  WK_CUDA_AT(cudaGetLastError(), "affine_stream_ader_kernel");
}

// compile-time TCK plans: the reference defaults (every_second reduction;
// ader_hdg with the shift, plain ader without)
template <int D, int N>
bool affine_stream_ader_launch(bool hdg, int stride, bool shift, const TckStreamArgs& a,
                               cudaStream_t s) {
  if constexpr (stream_ader_supported(D, N)) {
    if (stride == 2 && hdg && shift) {
      launch_stream_ader<D, N, true, 2, true>(a, s);
      return true;
    }
    if (stride == 2 && !hdg && !shift) {
      launch_stream_ader<D, N, false, 2, false>(a, s);
      return true;
    }
  }
  return false;
}

template <int D, int N>
void affine_ader_a_launch(bool cart, bool hdg, const TckArgs& a, cudaStream_t s) {
  if (cart && a.op.geo_class == nullptr) {
    if (hdg) return launch_group_ader<D, N, true>(a, s);
    return launch_group_ader<D, N, false>(a, s);
  }
  affine_ader_a_general_launch<D, N>(cart, hdg, a, s);
}

template <int N, int KIND, int STRIDE, bool SHIFT>
bool launch_curved_stream(const CurvedStreamArgs& a, cudaStream_t s) {
  using K = typename CurvedKernelCfg<N, KIND, STRIDE, SHIFT>::K;
  if constexpr (K::BYTES > 227 * 1024) {
    return false;
  } else {
    auto kern = curved_stream_kernel<N, KIND, STRIDE, SHIFT>;
    const int per_sm = resident_per_sm(kern, K::TG, K::BYTES);
    const long long tiles = a.t.op.E;
    if (tiles == 0) return true;
    const long long grid = std::min<long long>(tiles, persistent_slots(per_sm, a.t.op.grid_hold));
    kern<<<(unsigned)grid, K::TG, K::BYTES, s>>>(a);
    WK_CUDA_AT(cudaGetLastError(), "curved_stream_kernel");
    return true;
  }
}

// persistent curved kernels: operator modes, and ADER kernel A with the
// reference-default plans (every_second; ader_hdg with shift, ader without)
template <int D, int N>
bool curved_stream_launch(int kind, int stride, bool shift, const CurvedStreamArgs& a,
                          cudaStream_t s) {
  if constexpr (stream_curved_supported(D, N)) {
    switch (kind) {
      case OUT_MINVK: return launch_curved_stream<N, OUT_MINVK, 0, false>(a, s);
      case OUT_RHS: return launch_curved_stream<N, OUT_RHS, 0, false>(a, s);
      case OUT_LSRK: return launch_curved_stream<N, OUT_LSRK, 0, false>(a, s);
      case OUT_ADERB: return launch_curved_stream<N, OUT_ADERB, 0, false>(a, s);
      case kCurvedAderHdg:
        if (stride == 2 && shift) return launch_curved_stream<N, kCurvedAderHdg, 2, true>(a, s);
        break;
      case kCurvedAder:
        if (stride == 2 && !shift) return launch_curved_stream<N, kCurvedAder, 2, false>(a, s);
        break;
    }
  }
  return false;
}

template <int D, int N>
void curved_op_launch(int mode, const AffineArgs& a, const CurvedArgs& g, cudaStream_t s) {
  if constexpr (N <= 8) {
    switch (mode) {
      case OUT_MINVK: return launch_curved_op<D, N, OUT_MINVK>(a, g, s);
      case OUT_RHS: return launch_curved_op<D, N, OUT_RHS>(a, g, s);
      case OUT_LSRK: return launch_curved_op<D, N, OUT_LSRK>(a, g, s);
      case OUT_ADERB: return launch_curved_op<D, N, OUT_ADERB>(a, g, s);
      case OUT_K: return launch_curved_op<D, N, OUT_K>(a, g, s);
    }
    throw WkError(WK_EINVAL, "bad curved operator mode");
  } else {
    throw WkError(WK_EINVAL, "curved geometry supports degrees up to 7");
  }
}

template <int D, int N>
void curved_ader_a_launch(bool hdg, const TckArgs& a, const CurvedArgs& g, cudaStream_t s) {
  if constexpr (N <= 8) {
    if (hdg) return launch_curved_ader_a<D, N, true>(a, g, s);
    return launch_curved_ader_a<D, N, false>(a, g, s);
  } else {
    throw WkError(WK_EINVAL, "curved geometry supports degrees up to 7");
  }
}

template void affine_op_launch<WK_D, WK_N>(bool, int, const AffineArgs&, cudaStream_t);
template void affine_ader_a_launch<WK_D, WK_N>(bool, bool, const TckArgs&, cudaStream_t);
template bool affine_stream_ader_launch<WK_D, WK_N>(bool, int, bool, const TckStreamArgs&,
                                                    cudaStream_t);
template bool curved_stream_launch<WK_D, WK_N>(int, int, bool, const CurvedStreamArgs&,
                                               cudaStream_t);
template void curved_op_launch<WK_D, WK_N>(int, const AffineArgs&, const CurvedArgs&,
                                           cudaStream_t);
// one cluster of up to 16 CTAs (one per SM), every CTA holding its element
// range in shared memory for the whole run
template <int D, int N>
bool small_lsrk_launch(const SmallArgs& a0, cudaStream_t s, bool dry_run) {
  using K = SmallCfg<D, N>;
  if (a0.E <= 0 || a0.stages > kSmallMaxStages) return false;
  const int nc = (int)std::min<long long>(kSmallMaxCluster, a0.E);
  const int epc = (int)((a0.E + nc - 1) / nc);
  const size_t smem = K::bytes(epc);
  if (smem > 227 * 1024) return false;
  if (dry_run) return true;
  auto kern = small_lsrk_kernel<D, N>;
  KernelSetup& ks = ensure_smem(kern, smem);
  if (!ks.nonportable_cluster) {   // clusters of 16 CTAs (portable limit: 8)
    WK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    ks.nonportable_cluster = true;
  }
  SmallArgs a = a0;
  a.epc = epc;
  const int threads = (int)std::min<long long>(1024, ((long long)epc * K::NODES + 31) / 32 * 32);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nc, 1, 1);
  cfg.blockDim = dim3((unsigned)std::max(threads, 32), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)nc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  WK_CUDA_AT(cudaLaunchKernelEx(&cfg, kern, a), "small_lsrk_kernel");
  return true;
}

template bool small_lsrk_launch<WK_D, WK_N>(const SmallArgs&, cudaStream_t, bool);
template void curved_ader_a_launch<WK_D, WK_N>(bool, const TckArgs&, const CurvedArgs&,
                                               cudaStream_t);

}  // namespace wk
