// Persistent, TMA-streamed ADER kernel A for axis-aligned (Cartesian) affine
// cells with the Taylor loop specialised at COMPILE TIME
// (stepping.py:215-285, reduction_schedule kernels.py:286-302):
//   ader_hdg: W = M^{-1} K U,  V = U - dt W,  y = M^{-1} TCK_shift(W)
//   ader:     y = M^{-1} TCK(U)
//
// affine_group_ader_kernel (wk_group_ader.cuh) interprets the op program at
// run time: every 1-D matrix entry is a shared-memory load, every op a loop
// with run-time extents, and the element's bytes arrive with no prefetch.
// ncu at config 2 (k = 4) counted ~6300 warp instructions per element for
// ~440 warp-DFMAs.  Here the program (make_tck_plan, the same op list
// get_program builds) is a template parameter pack, so
//   * every 1-D matrix (S at each degree, projections, interpolations) and
//     every Taylor weight is a kernel parameter read as a constant-bank
//     operand of the DFMA — no load instruction at all;
//   * every op has compile-time extents (fully unrolled pencil / line loops);
//   * the accumulators live in REGISTERS with an element-wise (coalesced)
//     ownership: lane + j*TG over the contiguous tile, so ACC ops touch only
//     the current field in shared memory and need no barrier, and y leaves
//     with coalesced stores straight from the registers;
//   * the element tiles stream in like the LSRK stage kernel: persistent
//     CTAs, two stages, U by one cp.async.bulk (TMA) per tile, neighbour face
//     values by cp.async one tile ahead, ordered tile queue (wk_stream.cuh).
// Shared memory per group: two stages (U tile + face values) and one work
// tile; the stage holding U becomes the second work tile once V is written.
#pragma once
#include <utility>

#include "wk_stream.cuh"
#include "wk_tck.cuh"

namespace wk {

constexpr int kPlanOps = 48;
constexpr int kPlanTab = 768;

struct TckStep {
  int code, a0, a1, a2;
};
struct TckPlan {
  int n, tab_len;
  TckStep ops[kPlanOps];
};

// get_program (wk_abi.cu) restated as a constexpr function for affine cells
// (full degree in the GL basis): identical op order and table offsets, so the
// host's table blob and per-op weights serve both.  ACC_* / LOAD carry the
// slot DEGREE in a0 (get_program: the slot offset); S: a0 = points, a1 =
// table offset; RESIZE: a0 = from-points, a1 = to-points, a2 = table offset.
__host__ __device__ constexpr TckPlan make_tck_plan(int k, int stride, bool shift) {
  TckPlan p{};
  bool has[16] = {};
  int n = 0, tab = 0;
  p.ops[n++] = TckStep{TCK_ACC_SET, k, k + 1, 0};
  has[k] = true;
  const int n_apps = shift ? (k - 1 > 0 ? k - 1 : 0) : k + 1;
  int deg = k, sdeg = k;
  for (int j = 1; j <= n_apps; ++j) {
    const int din = sdeg;
    const int dout = (stride && j % stride == 0) ? (sdeg - stride > 0 ? sdeg - stride : 0) : sdeg;
    sdeg = dout;
    if (din == 0) break;
    p.ops[n++] = TckStep{TCK_S, deg + 1, tab, 0};
    tab += (deg + 1) * (deg + 1);
    if (dout != din) {
      p.ops[n++] = TckStep{TCK_RESIZE, deg + 1, dout + 1, tab};
      tab += (dout + 1) * (deg + 1);
      deg = dout;
    }
    if (has[deg]) {
      p.ops[n++] = TckStep{TCK_ACC_ADD, deg, deg + 1, 0};
    } else {
      has[deg] = true;
      p.ops[n++] = TckStep{TCK_ACC_SET, deg, deg + 1, 0};
    }
  }
  for (int lo = 0; lo < k; ++lo) {
    if (!has[lo]) continue;
    int hi = lo + 1;
    while (!has[hi]) ++hi;
    p.ops[n++] = TckStep{TCK_LOAD, lo, lo + 1, 0};
    p.ops[n++] = TckStep{TCK_RESIZE, lo + 1, hi + 1, tab};
    tab += (hi + 1) * (lo + 1);
    p.ops[n++] = TckStep{TCK_ACC_ADD, hi, hi + 1, 0};
  }
  p.n = n;
  p.tab_len = tab;
  return p;
}

struct TckStreamArgs {
  AffineArgs op;           // operator inputs (u = U), geometry, material, tile queue
  double* y;               // M^{-1} T (GL coefficients)
  double* v_out;           // ader_hdg: V = U - dt W
  double dt;
  double w[kPlanOps];      // per-op weight (Taylor weight or 1)
  double tab[kPlanTab];    // the plan's 1-D matrices, get_program's blob
};

template <int D, int N>
struct StreamAderCfg {
  using G = GroupCfg<D, N>;
  static constexpr int C = D + 1, NODES = G::NODES, NF = G::NF, EPG = G::EPG;
  static constexpr int PW = G::TG;                       // pencil lanes
  // lanes per pencil: 1 (the lane finishes v_m and its p share) for n <= 6;
  // 2 for n >= 7 (half 0: v_m, half 1: p share), which halves the
  // element-wise registers per lane (accumulators) of the large tiles
#ifndef WK_ADER_H2_MIN_N
#define WK_ADER_H2_MIN_N 7
#endif
  static constexpr int H = N >= WK_ADER_H2_MIN_N ? 2 : 1;
  static constexpr int TG = H * PW;
  static constexpr int TILE = EPG * C * NODES;
  static constexpr int NBF = EPG * D * 2 * 2 * NF;      // [q][m][side][v_m,p][fn]
  static constexpr int BUF = (TILE + NBF + 1) / 2 * 2;   // one stage: U tile | faces
  static constexpr int OFF_W = 2 * BUF;                  // work tile (W, p partials in place)
  static constexpr int OFF_MAT = (OFF_W + TILE + 1) / 2 * 2;
  static constexpr int OFF_BAR = OFF_MAT + EPG * 4;
  static constexpr int OFF_Q = OFF_BAR + 2;             // two 8-byte mbarriers
  static constexpr int OFF_GEO = OFF_Q + 4;             // two tile-queue slots + elements
  static constexpr int TOTAL = OFF_GEO + GeoLayout<D>::STRIDE;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  static constexpr bool TILE16 = (TILE * 8) % 16 == 0;
  static constexpr int RPL = (TILE + TG - 1) / TG;      // element-wise values per lane
  // an explicit minimum of one CTA per SM changes ptxas's scheduling: 2 %
  // faster at n <= 6 (configs 2, 5), 6 % slower at n = 8 (config 4), where 0
  // (no minimum) keeps the default
#ifndef WK_ADER_MINB
#define WK_ADER_MINB (N <= 6 ? 1 : (N == 8 ? 3 : 0))
#endif
  static constexpr int MINB = WK_ADER_MINB;
};

// run-time eligibility of the compile-time plans instantiated in wk_inst.cu
__host__ __device__ constexpr bool stream_ader_supported(int D, int N) {
  return (D == 2 || D == 3) && N >= 2 && N <= 9;
}

namespace sader {

template <int D, int NN>
__device__ __forceinline__ constexpr int npts() {
  return D == 3 ? NN * NN * NN : NN * NN;
}

// S on a Cartesian cell at NN points per direction (operator.py:286-306):
// v_m <- (ir G_mm) D p along m,  p <- sum_m (c2r G_mm) D v_m; lane = pencil,
// the p shares accumulate in place in nxt's p component.
template <int D, int N, int NN, int TOFF>
__device__ __forceinline__ void apply_S1(const TckStreamArgs& T, const double* cur, double* nxt,
                                        const double* smat, const double* geo, int lane) {
  using K = StreamAderCfg<D, N>;
  constexpr int C = K::C, NODES = K::NODES, EPG = K::EPG, TG = K::TG;
  constexpr int NNF = D == 3 ? NN * NN : NN;
  constexpr int ITEMS = EPG * NNF;
  constexpr int NIT = (ITEMS + TG - 1) / TG;
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? NN : NN * NN);
    const double gmm = geo[m * D + m];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int t = lane + it * TG;
      if (ITEMS % TG == 0 || t < ITEMS) {
        const int qq = t / NNF, ln = t - (t / NNF) * NNF;
        const int b0 = m == 0 ? ln * NN : (m == 1 ? ln % NN + (ln / NN) * NN * NN : ln);
        const double* src = cur + qq * C * NODES + b0;
        double xp[NN], xv[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) {
          xp[j] = src[D * NODES + j * sm];
          xv[j] = src[m * NODES + j * sm];
        }
        const double cv = smat[qq * 4 + 0] * gmm, cp = smat[qq * 4 + 1] * gmm;
        double* dst = nxt + qq * C * NODES + b0;
#pragma unroll
        for (int i = 0; i < NN; ++i) {
          double av = 0.0, ap = 0.0;
#pragma unroll
          for (int j = 0; j < NN; ++j) {
            const double d = T.tab[TOFF + i * NN + j];
            av = fma(d, xp[j], av);
            ap = fma(d, xv[j], ap);
          }
          av *= cv;
          ap *= cp;
          dst[m * NODES + i * sm] = av;
          if (m == 0) dst[D * NODES + i * sm] = ap;
          else dst[D * NODES + i * sm] += ap;
        }
      }
    }
    group_sync<TG>(0);
  }
}

// S on a Cartesian cell at NN points per direction (operator.py:286-306):
// v_m <- (ir G_mm) D p along m,  p <- sum_m (c2r G_mm) D v_m.  Two lanes per
// pencil: half 0 differentiates p into v_m, half 1 differentiates v_m into
// its p share, accumulated in place in nxt's p component.
template <int D, int N, int NN, int TOFF>
__device__ __forceinline__ void apply_S2(const TckStreamArgs& T, const double* cur, double* nxt,
                                        const double* smat, const double* geo, int lane) {
  using K = StreamAderCfg<D, N>;
  constexpr int C = K::C, NODES = K::NODES, EPG = K::EPG, TG = K::TG;
  constexpr int NNF = D == 3 ? NN * NN : NN;
  constexpr int ITEMS = EPG * NNF;
  constexpr int NIT = (2 * ITEMS + TG - 1) / TG;
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? NN : NN * NN);
    const double gmm = geo[m * D + m];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int t = lane + it * TG;
      if ((2 * ITEMS) % TG == 0 || t < 2 * ITEMS) {
        const int half = t >= ITEMS ? 1 : 0;
        const int tt = t - half * ITEMS;
        const int qq = tt / NNF, ln = tt - (tt / NNF) * NNF;
        const int b0 = m == 0 ? ln * NN : (m == 1 ? ln % NN + (ln / NN) * NN * NN : ln);
        const double* src = cur + qq * C * NODES + (half ? m : D) * NODES + b0;
        double x[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) x[j] = src[j * sm];
        const double coef = smat[qq * 4 + half] * gmm;   // ir (v) or c2r (p)
        double* dst = nxt + qq * C * NODES + (half ? D : m) * NODES + b0;
#pragma unroll
        for (int i = 0; i < NN; ++i) {
          double a = 0.0;
#pragma unroll
          for (int j = 0; j < NN; ++j) a = fma(T.tab[TOFF + i * NN + j], x[j], a);
          a *= coef;
          if (half == 0 || m == 0) dst[i * sm] = a;
          else dst[i * sm] += a;
        }
      }
    }
    group_sync<TG>(0);
  }
}

// S at the full degree of a 3-D n = 8 element on the FP64 TENSOR CORES
// (mma.sync m8n8k4 f64, DMMA): per direction, Y = D X for the 64 pencils of
// p (-> v_m) and of v_m (-> the p share) as 16 chunks of 8 pencils, two
// k-steps each (n = 8 = 2 x 4: no padding), the 8 x 8 derivative matrix held
// as two A fragments per lane for the whole op.  A warp instruction does 256
// FMAs where the CUDA-core pencil version issues one DFMA per 32; the S ops
// at degree 7 are ~3/4 of config 4's kernel-A FLOPs (ncu: issue/latency
// bound at 26 % of the FP64 pipe with 255 registers).  Fragment layout
// (tools/dmma_check.cu): A lane l = M[l>>2][l&3], B lane l = X[l&3][l>>2],
// C lane l = Y[l>>2][2(l&3)+{0,1}].  Chunks of 8 pencils are affine in
// memory for every direction, so the fragment addresses need no division.
template <int D, int N, int TOFF>
__device__ __forceinline__ void apply_S_mma8(const TckStreamArgs& T, const double* cur,
                                             double* nxt, const double* smat, const double* geo,
                                             int lane) {
  using K = StreamAderCfg<D, N>;
  constexpr int NODES = K::NODES, TG = K::TG, NW = TG / 32;
  const int l32 = lane & 31, warp = lane >> 5;
  const int ar = l32 >> 2, ac = l32 & 3;
  const double a0 = T.tab[TOFF + ar * 8 + ac], a1 = T.tab[TOFF + ar * 8 + 4 + ac];
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? 8 : 64);
    const int ps = m == 0 ? 8 : 1;            // stride between a chunk's pencils
    const double gmm = geo[m * D + m];
    const double cv = smat[0] * gmm, cp = smat[1] * gmm;
#pragma unroll
    for (int uu = 0; uu < 16 / NW; ++uu) {    // 8 chunks x {p -> v_m, v_m -> p}
      const int u = warp + uu * NW;
      const int half = u >> 3, c = u & 7;
      const int cb = m == 2 ? 8 * c : 64 * c;
      const double* src = cur + (half ? m : D) * NODES + cb;
      const int bo = ar * ps + ac * sm;
      double c0 = 0.0, c1 = 0.0;
      dmma884(c0, c1, a0, src[bo]);
      dmma884(c0, c1, a1, src[bo + 4 * sm]);
      const int n0 = cb + (2 * ac) * ps + ar * sm;
      const int n1 = n0 + ps;
      if (!half) {
        nxt[m * NODES + n0] = c0 * cv;
        nxt[m * NODES + n1] = c1 * cv;
      } else if (m == 0) {
        nxt[D * NODES + n0] = c0 * cp;
        nxt[D * NODES + n1] = c1 * cp;
      } else {
        nxt[D * NODES + n0] += c0 * cp;
        nxt[D * NODES + n1] += c1 * cp;
      }
    }
    group_sync<TG>(0);
  }
}

template <int D, int N, int NN, int TOFF>
__device__ __forceinline__ void apply_S(const TckStreamArgs& T, const double* cur, double* nxt,
                                        const double* smat, const double* geo, int lane) {
#ifndef WK_ADER_DMMA
#define WK_ADER_DMMA 1
#endif
  if constexpr (WK_ADER_DMMA && D == 3 && N == 8 && NN == 8 && StreamAderCfg<D, N>::EPG == 1)
    apply_S_mma8<D, N, TOFF>(T, cur, nxt, smat, geo, lane);
  else if constexpr (StreamAderCfg<D, N>::H == 2) apply_S2<D, N, NN, TOFF>(T, cur, nxt, smat, geo, lane);
  else apply_S1<D, N, NN, TOFF>(T, cur, nxt, smat, geo, lane);
}

// projection / interpolation NF_ -> NT_ points in every direction
// (operator.py:308-325); result ends in cur
template <int D, int N, int TG, int EPG, int NF_, int NT_, int TOFF>
__device__ __forceinline__ void resize(const TckStreamArgs& T, double*& cur, double*& nxt,
                                       int lane) {
  constexpr int C = D + 1, NODES = D == 3 ? N * N * N : N * N;
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const int lo_ext = m == 0 ? 1 : (m == 1 ? NT_ : NT_ * NT_);
    const int hi_ext = D == 3 ? (m == 0 ? NF_ * NF_ : (m == 1 ? NF_ : 1)) : (m == 0 ? NF_ : 1);
    const int lines = lo_ext * hi_ext;
    const int items = EPG * C * lines;
    constexpr int MAXL = D == 3 ? (NF_ > NT_ ? NF_ : NT_) * (NF_ > NT_ ? NF_ : NT_) : (NF_ > NT_ ? NF_ : NT_);
    constexpr int NIT = (EPG * C * MAXL + TG - 1) / TG;
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int t = lane + it * TG;
      if (t < items) {
        const int qc = t / lines, l = t - (t / lines) * lines;
        const int hi = l / lo_ext, lo = l - (l / lo_ext) * lo_ext;
        const double* src = cur + qc * NODES + lo + hi * lo_ext * NF_;
        double x[NF_];
#pragma unroll
        for (int j = 0; j < NF_; ++j) x[j] = src[j * lo_ext];
        double* dst = nxt + qc * NODES + lo + hi * lo_ext * NT_;
#pragma unroll
        for (int i = 0; i < NT_; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < NF_; ++j) acc = fma(T.tab[TOFF + i * NF_ + j], x[j], acc);
          dst[i * lo_ext] = acc;
        }
      }
    }
    group_sync<TG>(0);
    double* tt = cur;
    cur = nxt;
    nxt = tt;
  }
}

// element-wise accumulator op on the degree-Q field in cur (ownership lane + j*TG)
template <int D, int N, int TG, int EPG, int Q, int CODE, int WI, int RPL>
__device__ __forceinline__ void acc_op(const TckStreamArgs& T, double (&acc)[RPL], double* cur,
                                       int lane) {
  constexpr int NODES = D == 3 ? N * N * N : N * N;
  constexpr int NP = npts<D, Q + 1>();
  constexpr int ITEMS = EPG * (D + 1) * NP;
  constexpr int NIT = (ITEMS + TG - 1) / TG;
  if (CODE == TCK_LOAD) group_sync<TG>(0);   // earlier readers of cur are done
#pragma unroll
  for (int j = 0; j < NIT; ++j) {
    const int f = lane + j * TG;
    if (ITEMS % TG == 0 || f < ITEMS) {
      const int qc = f / NP, pt = f - (f / NP) * NP;
      double* cv = cur + qc * NODES + pt;
      if (CODE == TCK_ACC_SET) acc[j] = T.w[WI] * *cv;
      else if (CODE == TCK_ACC_ADD) acc[j] = acc[j] + T.w[WI] * *cv;
      else *cv = acc[j];
    }
  }
  if (CODE == TCK_LOAD) group_sync<TG>(0);
}

template <int D, int N, int STRIDE, bool SHIFT>
struct Plan {
  static constexpr TckPlan P = make_tck_plan(N - 1, STRIDE, SHIFT);
};

// op I of the plan (compile time)
template <int D, int N, int STRIDE, bool SHIFT, int I>
__device__ __forceinline__ void run_op(const TckStreamArgs& T, double*& cur, double*& nxt,
                                       double (&acc)[N][StreamAderCfg<D, N>::RPL],
                                       const double* smat, const double* geo, int lane) {
  constexpr TckStep op = Plan<D, N, STRIDE, SHIFT>::P.ops[I];
  if constexpr (op.code == TCK_S) {
    apply_S<D, N, op.a0, op.a1>(T, cur, nxt, smat, geo, lane);
    double* tt = cur;
    cur = nxt;
    nxt = tt;
  } else if constexpr (op.code == TCK_RESIZE) {
    resize<D, N, StreamAderCfg<D, N>::TG, StreamAderCfg<D, N>::EPG, op.a0, op.a1, op.a2>(
        T, cur, nxt, lane);
  } else {
    acc_op<D, N, StreamAderCfg<D, N>::TG, StreamAderCfg<D, N>::EPG, op.a0, op.code, I>(
        T, acc[op.a0], cur, lane);
  }
}

template <int D, int N, int STRIDE, bool SHIFT, int... I>
__device__ __forceinline__ void run_plan(const TckStreamArgs& T, double*& cur, double*& nxt,
                                         double (&acc)[N][StreamAderCfg<D, N>::RPL],
                                         const double* smat, const double* geo, int lane,
                                         std::integer_sequence<int, I...>) {
  (run_op<D, N, STRIDE, SHIFT, I>(T, cur, nxt, acc, smat, geo, lane), ...);
}

}  // namespace sader

template <int D, int N, bool HDG, int STRIDE, bool SHIFT>
__global__ void __launch_bounds__(StreamAderCfg<D, N>::TG, StreamAderCfg<D, N>::MINB)
affine_stream_ader_kernel(const __grid_constant__ TckStreamArgs T) {
  using K = StreamAderCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, EPG = K::EPG, TG = K::TG;
  constexpr int RPL = K::RPL;
  constexpr TckPlan PLAN = sader::Plan<D, N, STRIDE, SHIFT>::P;
  extern __shared__ __align__(128) double smem[];
  double* const sW = smem + K::OFF_W;
  double* const smat = smem + K::OFF_MAT;
  unsigned long long* const bar = reinterpret_cast<unsigned long long*>(smem + K::OFF_BAR);
  double* const geo = smem + K::OFF_GEO;
  const int lane = threadIdx.x;
  WK_CHECK_SMEM(K::BYTES);
  const double* const gU = T.op.u;
  const int* const gnbr = T.op.nbr;
  const double* const gghost = T.op.ghost;
  const double* const gmat = T.op.mat;
  unsigned* const sched = T.op.sched;
  const bool has_ghost = T.op.has_ghost != 0;
  const bool stab = T.op.stab != 0;
  const double dt = T.dt;
  for (int i = lane; i < GLy::STRIDE; i += TG) geo[i] = T.op.geo[i];
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  group_sync<TG>(0);

  const long long e_begin = T.op.e_begin;
  const long long e_end = e_begin + T.op.E;
  const long long ntiles = (T.op.E + EPG - 1) / EPG;
  const bool tma = K::TILE16 && (((e_begin * C * NODES) & 1) == 0);
  constexpr int PW = K::PW;
  const int half = K::H == 2 ? lane / PW : 0, pl_ = lane - half * PW;
  const int q = pl_ / NF, fn = pl_ - (pl_ / NF) * NF;
  const bool plane_lane = pl_ < EPG * NF;

  long long tile = blockIdx.x;   // grid <= ntiles (launcher)
  int noff[D][2];
#pragma unroll
  for (int m = 0; m < D; ++m)
#pragma unroll
    for (int s = 0; s < 2; ++s) noff[m][s] = face_to_node<N>(m, 1 - s, fn);
  unsigned nb_u32[2];
#pragma unroll
  for (int b = 0; b < 2; ++b)
    nb_u32[b] = smem_u32(smem + b * K::BUF + K::TILE + (q * D * 2 * 2) * NF + fn);

  auto fetch_ids = [&](long long t, long long et, int (&ids)[2 * D]) {
    const long long e = et + q;
#pragma unroll
    for (int f = 0; f < 2 * D; ++f)
      ids[f] = (HDG && plane_lane && t < ntiles && e < e_end) ? __ldg(gnbr + e * 2 * D + f) : -1;
  };
  auto fetch_mat = [&](long long t, long long et, double (&mt)[4]) {
    const long long e = et + q;
    const bool ok = plane_lane && t < ntiles && e < e_end;
#pragma unroll
    for (int i = 0; i < 4; ++i) mt[i] = ok ? __ldg(gmat + e * kMatStride + i) : 0.0;
  };
  auto issue = [&](long long et, int b, const int (&ids)[2 * D]) {
    const long long e0 = et;
    const int nel = (int)min((long long)EPG, e_end - e0);
    double* su = smem + b * K::BUF;
    const unsigned bytes = (unsigned)(nel * C * NODES * 8);
    const double* gu = gU + e0 * C * NODES;
    if (tma && (bytes % 16) == 0) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&bar[b], bytes);
        bulk_g2s(su, gu, bytes, &bar[b]);
      }
    } else {
      for (int i = lane; i < nel * C * NODES; i += TG) cp_async8(su + i, gu + i);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar[b]))
                     : "memory");
      }
    }
    if (HDG && plane_lane && q < nel) {
      // H == 2: half 0 gathers the neighbours' v_m, half 1 their p
      const unsigned dst = nb_u32[b] + (unsigned)(half * NF) * 8u;
#pragma unroll
      for (int m = 0; m < D; ++m)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int nb = ids[2 * m + s];
          WK_CHECK_NBR(T.op, nb);
          const unsigned d0 = dst + (unsigned)(((m * 2 + s) * 2) * NF) * 8u;
#pragma unroll
          for (int h = 0; h < 3 - K::H; ++h) {
            const int comp = (K::H == 2 ? half : h) ? D : m;
            const unsigned dd = d0 + (unsigned)(h * NF) * 8u;
            if (nb >= 0) {
              cp_async8_u32(dd, gU + (long long)nb * (C * NODES) + noff[m][s] + comp * NODES);
            } else if (has_ghost && nb <= -2) {
              cp_async8_u32(dd, gghost + (long long)ghost_slot(nb) * C * NF + fn + comp * NF);
            }
          }
        }
    }
  };

  int ids_cur[2 * D], ids_nxt[2 * D], ids_nn[2 * D];
  double mat_cur[4], mat_nxt[4];
  long long e_tile = tile_elem<EPG>(T.op, tile);
  fetch_ids(tile, e_tile, ids_cur);
  fetch_mat(tile, e_tile, mat_cur);
  issue(e_tile, 0, ids_cur);
  cp_async_commit();

  // ordered tile queue (see affine_stream_kernel)
  long long* const qslot = reinterpret_cast<long long*>(smem + K::OFF_Q);
  const long long kNone = ntiles;
  const long long dyn0 = 2LL * gridDim.x;
  const unsigned qcap = (unsigned)(ntiles + 4LL * gridDim.x + 64);   // > any claim count
  long long nxt = tile + gridDim.x < ntiles ? tile + gridDim.x : kNone;
  long long e_nxt = nxt < ntiles ? tile_elem<EPG>(T.op, nxt) : 0;
  unsigned raw = 0;
  bool pend = false;
  if (lane == 0) {
    long long w = kNone;
    if (nxt < ntiles) {
      w = dyn0 + (long long)atomic_claim(sched, qcap);
      if (w >= ntiles) w = kNone;
    }
    qslot[1] = w;
    qslot[3] = w < ntiles ? tile_elem<EPG>(T.op, w) : 0;   // its first element
    pend = w < ntiles;
    if (pend) raw = atomic_claim(sched, qcap);
  }
  group_sync<TG>(0);
  long long nn = qslot[1], e_nn = qslot[3];
  fetch_ids(nxt, e_nxt, ids_nxt);
  int buf = 0;
  unsigned it = 0;
  while (tile < ntiles) {
    if (nxt < ntiles) issue(e_nxt, buf ^ 1, ids_nxt);
    cp_async_commit();
    fetch_ids(nn, e_nn, ids_nn);
    fetch_mat(nxt, e_nxt, mat_nxt);
    if (tma && T.op.l2pf && lane == 0 && nn < ntiles) {
      const long long e2 = e_nn;
      const unsigned b2 = (unsigned)(min((long long)EPG, e_end - e2) * C * NODES * 8) & ~15u;
      bulk_prefetch_l2(gU + e2 * C * NODES, b2);
    }
    if (lane == 0) {
      long long w = kNone;
      if (pend) {
        w = dyn0 + (long long)raw;
        if (w >= ntiles) w = kNone;
      }
      qslot[it & 1] = w;
      qslot[2 + (it & 1)] = w < ntiles ? tile_elem<EPG>(T.op, w) : 0;
      pend = w < ntiles;
      if (pend) raw = atomic_claim(sched, qcap);
    }
    const long long e0 = e_tile;
    const int nel = (int)min((long long)EPG, e_end - e0);
    const int nvals = nel * C * NODES;
    const long long goff = e0 * C * NODES;
    if (half == 0 && plane_lane && fn == 0 && q < nel) {
#pragma unroll
      for (int i = 0; i < 4; ++i) smat[q * 4 + i] = mat_cur[i];
    }
    mbar_wait(&bar[buf], (it >> 1) & 1u);
    cp_async_wait<1>();
    group_sync<TG>(0);
    const long long nnn = qslot[it & 1], e_nnn = qslot[2 + (it & 1)];

    double* su = smem + buf * K::BUF;
    double* cur;
    double* nx;
    if constexpr (HDG) {
      if constexpr (K::H == 1) {
      // ---- W = M^{-1} K U into sW (wk_stream.cuh's sweeps) -----------------
      const double* snb = su + K::TILE;
      const bool plane = plane_lane && q < nel;
      const double ir = mat_cur[0], c2r = mat_cur[1], tau = plane ? mat_cur[2] : 1.0,
                   irt = mat_cur[3];
#pragma unroll
      for (int m = 0; m < D; ++m) {
        const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
        if (plane) {
          const int nb0 = pencil_base<N>(m, fn);
          const double* ul = su + q * C * NODES + nb0;
          double* fl = sW + q * C * NODES + nb0;
          double pl[N], vl[N];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            pl[i] = ul[D * NODES + i * sm];
            vl[i] = ul[m * NODES + i * sm];
          }
          double fv0, fp0, fv1, fp1;
          const double* f0 = snb + (((q * D + m) * 2 + 0) * 2) * NF + fn;
          const double* f1 = snb + (((q * D + m) * 2 + 1) * 2) * NF + fn;
          const bool w0 = ids_cur[2 * m] == -1, w1 = ids_cur[2 * m + 1] == -1;
          cart_face_flux(vl[0], pl[0], w0 ? vl[0] : f0[0], w0 ? -pl[0] : f0[NF],
                         geo[GLy::NORMAL + (m * 2 + 0) * D + m], geo[GLy::FSCALE + m * 2 + 0],
                         ir, c2r, tau, irt, stab, fv0, fp0);
          cart_face_flux(vl[N - 1], pl[N - 1], w1 ? vl[N - 1] : f1[0], w1 ? -pl[N - 1] : f1[NF],
                         geo[GLy::NORMAL + (m * 2 + 1) * D + m], geo[GLy::FSCALE + m * 2 + 1],
                         ir, c2r, tau, irt, stab, fv1, fp1);
          const double gmm = geo[m * D + m];
          const double cv = ir * gmm, cp = c2r * gmm;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double ap = 0.0, av = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) {
              const double a = T.op.cA[i * N + j];
              ap = fma(a, pl[j], ap);
              av = fma(a, vl[j], av);
            }
            const double l0 = T.op.cL0[i], l1 = T.op.cL1[i];
            fl[m * NODES + i * sm] = fma(cv, ap, fma(l0, fv0, l1 * fv1));
            double resp = fma(cp, av, fma(l0, fp0, l1 * fp1));
            if (m > 0) resp += fl[D * NODES + i * sm];
            fl[D * NODES + i * sm] = resp;
          }
        }
        group_sync<TG>(0);
      }
      } else {
      // ---- W = M^{-1} K U into sW (wk_stream.cuh's sweeps, two lanes per
      //      pencil: half 0 finishes v_m, half 1 accumulates p) --------------
      const double* snb = su + K::TILE;
      const bool plane = plane_lane && q < nel;
      const double ir = mat_cur[0], c2r = mat_cur[1], tau = plane ? mat_cur[2] : 1.0,
                   irt = mat_cur[3];
#pragma unroll
      for (int m = 0; m < D; ++m) {
        const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
        if (plane) {
          const int nb0 = pencil_base<N>(m, fn);
          const double* ul = su + q * C * NODES + nb0;
          double* fl = sW + q * C * NODES + nb0;
          double x[N];
#pragma unroll
          for (int i = 0; i < N; ++i) x[i] = ul[(half ? m : D) * NODES + i * sm];
          // own traces at both ends (the other half's line endpoints)
          const double o0 = ul[(half ? D : m) * NODES], o1 = ul[(half ? D : m) * NODES + (N - 1) * sm];
          const double vo0 = half ? x[0] : o0, po0 = half ? o0 : x[0];
          const double vo1 = half ? x[N - 1] : o1, po1 = half ? o1 : x[N - 1];
          double fv0, fp0, fv1, fp1;
          const double* f0 = snb + (((q * D + m) * 2 + 0) * 2) * NF + fn;
          const double* f1 = snb + (((q * D + m) * 2 + 1) * 2) * NF + fn;
          const bool w0 = ids_cur[2 * m] == -1, w1 = ids_cur[2 * m + 1] == -1;
          cart_face_flux(vo0, po0, w0 ? vo0 : f0[0], w0 ? -po0 : f0[NF],
                         geo[GLy::NORMAL + (m * 2 + 0) * D + m], geo[GLy::FSCALE + m * 2 + 0],
                         ir, c2r, tau, irt, stab, fv0, fp0);
          cart_face_flux(vo1, po1, w1 ? vo1 : f1[0], w1 ? -po1 : f1[NF],
                         geo[GLy::NORMAL + (m * 2 + 1) * D + m], geo[GLy::FSCALE + m * 2 + 1],
                         ir, c2r, tau, irt, stab, fv1, fp1);
          const double gmm = geo[m * D + m];
          const double coef = (half ? c2r : ir) * gmm;
          const double g0 = half ? fp0 : fv0, g1 = half ? fp1 : fv1;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double a = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) a = fma(T.op.cA[i * N + j], x[j], a);
            double res = fma(coef, a, fma(T.op.cL0[i], g0, T.op.cL1[i] * g1));
            if (half == 0) {
              fl[m * NODES + i * sm] = res;
            } else {
              if (m > 0) res += fl[D * NODES + i * sm];
              fl[D * NODES + i * sm] = res;
            }
          }
        }
        group_sync<TG>(0);
      }
      }
      // ---- V = U - dt W (coalesced) ------------------------------------------
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        const int idx = lane + j * TG;
        if (idx < nvals) __stcs(T.v_out + goff + idx, su[idx] - dt * sW[idx]);   // streamed: evict first
      }
      group_sync<TG>(0);   // U is dead: its stage becomes the second work tile
      cur = sW;
      nx = su;
    } else {
      cur = su;
      nx = sW;
    }

    // ---- the Taylor loop, compile-time plan ----------------------------------
    double acc[N][RPL];
    sader::run_plan<D, N, STRIDE, SHIFT>(T, cur, nx, acc, smat, geo, lane,
                                        std::make_integer_sequence<int, PLAN.n>{});
    // y = acc_k, straight from the registers
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
      const int idx = lane + j * TG;
      if (idx < nvals) __stcs(T.y + goff + idx, acc[N - 1][j]);
    }
    group_sync<TG>(0);   // stage, work tile and smat free for the next tile
#pragma unroll
    for (int f = 0; f < 2 * D; ++f) {
      ids_cur[f] = ids_nxt[f];
      ids_nxt[f] = ids_nn[f];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) mat_cur[i] = mat_nxt[i];
    buf ^= 1;
    ++it;
    tile = nxt;
    nxt = nn;
    nn = nnn;
    e_tile = e_nxt;
    e_nxt = e_nn;
    e_nn = e_nnn;
  }
  sched_done(sched, lane == 0, pend, raw);
}

}  // namespace wk
