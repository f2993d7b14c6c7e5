// Persistent, TMA-streamed kernels for curved (per-point metric) 3-D cells:
// the fused operator (LSRK stage, rhs, M^{-1}K, ADER kernel B) and ADER
// kernel A with the compile-time Taylor plan (wk_stream_ader.cuh).
//
// Arithmetic: the reference's quadrature split form (operator.py:149-246)
// with the GeometryCache arrays (mesh.py:162-188), fused with the inverse
// mass, M^{-1}K = B^{-1}(x)3 [R/JxW] (operator.py:250-258; wk_curved.cuh has
// the derivation).  The work is organised in DIRECTIONAL LINE TASKS:
//
//   every metric term of the split form couples the field only along one
//   reference direction m at a time: the strong half at a Gauss point is
//   sum_m G_mi d_m p (resp. sum_{m,i} G_mi d_m v_i), the weak half is
//   sum_m D_m^T [G_m. flux] and the face lift of faces (m,0), (m,1) acts along
//   m.  So the quadrature-space residual splits into three partial tiles
//   R = R_0 + R_1 + R_2, and R_m is produced by independent tasks
//   (m, line along m, component), each holding its line in registers:
//     v_c task: p line -> D p -> 1/2 ir JxW G_mc D p  +  D^T(-1/2 ir JxW G_mc p)
//     p task:   v_0..2 lines -> sum_c 1/2 c2r JxW G_mc D v_c  +  D^T(weak flux)
//     both:     + the two face lifts (rows 0 and n-1 of B^{-1}) at the line ends.
//   The 1-D matrices are kernel parameters with compile-time indices (DFMA
//   constant-bank operands, no loads), every task does n^2 FMAs per n loads.
//   The own face traces come from the Gauss values by the same endpoint rows
//   of B^{-1} (exact: the trace of a degree-k polynomial), so only the
//   neighbours' GL face nodes need the 2-D B sweeps.
//   The ADER S operator (operator.py:286-306) uses the same split: three
//   partial tiles, summed by the accumulator op that consumes them.
//
// Per element: 3 sweep phases (GL -> Gauss, neighbour traces alongside), the
// face-integrand phase, ONE line-task phase and 3 B^{-1} sweeps: 8 barriers
// for the operator (the per-point formulation needed 19).
//
// Streaming: persistent CTAs on the ordered tile queue (wk_stream.cuh).  The
// U tile is double-buffered (one cp.async.bulk per tile); the metric arrays
// (inverse Jacobian and JxW at the Gauss points, face normals and face JxW,
// the reduced-degree metrics of the Taylor plan) and the neighbour face
// values are SINGLE-buffered: the next element's copies are issued as soon as
// the current element's last reader is done (after the line tasks; for ADER
// kernel A after the plan's last S), which keeps the operator kernel at three
// CTAs per SM at n = 6 (config 3).
#pragma once
#include "wk_curved.cuh"
#include "wk_stream_ader.cuh"

namespace wk {

constexpr int kCTab = 5 * kMaxN * kMaxN;

// Per-element metric record (built once at context creation from the
// GeometryCache arrays, wk_abi.cu): inv_jac | JxW | face normals | face JxW at
// the degree-k points, contiguous per element so ONE cp.async.bulk stages it.
template <int N>
struct CRec {
  static constexpr int NODES = N * N * N, NF = N * N;
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  static constexpr int IJ = 0;
  static constexpr int JW = IJ + ev(9 * NODES);
  static constexpr int FN = JW + ev(NODES);
  static constexpr int FJ = FN + ev(6 * 3 * NF);
  static constexpr int LEN = FJ + ev(6 * NF);
};
inline int crec_len(int n) {
  const int nodes = n * n * n, nf = n * n;
  auto ev = [](int x) { return (x + 1) / 2 * 2; };
  return ev(9 * nodes) + ev(nodes) + ev(18 * nf) + ev(6 * nf);
}

struct CurvedStreamArgs {
  TckStreamArgs t;                 // t.op: operator inputs / outputs, tile queue; t.w, t.tab: plan
  const double* rec;               // (E, CRec<n>::LEN) metric records
  const double* inv_jac[kMaxN];    // [q]: (E, d, d, (q+1)^d) at the degree-q Gauss points
  const double* jxw;               // (E, n^d) at the degree-k Gauss points
  const double* fnormal[6];        // (E, d, n^{d-1}) per face 2m+s
  const double* fjxw[6];           // (E, n^{d-1})
  double ctab[kCTab];              // B | B^{-1} | D_co | D_co^T | B^T, n x n each
};

__host__ __device__ constexpr bool stream_curved_supported(int D, int N) {
  return D == 3 && N >= 2 && N <= 7;   // n = 8 tiles exceed shared memory
}

// reduced metric degrees (< k) read by a plan's S ops, staged per element
__host__ __device__ constexpr bool plan_uses_S(const TckPlan& p, int q) {
  for (int i = 0; i < p.n; ++i)
    if (p.ops[i].code == TCK_S && p.ops[i].a0 == q + 1) return true;
  return false;
}
__host__ __device__ constexpr int red_off(const TckPlan& p, int k, int q) {
  int off = 0;
  for (int r = 0; r < q && r < k; ++r)
    if (plan_uses_S(p, r)) off += (9 * (r + 1) * (r + 1) * (r + 1) + 1) / 2 * 2;
  return off;
}
__host__ __device__ constexpr int red_len(const TckPlan& p, int k) { return red_off(p, k, k); }
__host__ __device__ constexpr int last_S(const TckPlan& p) {
  int l = -1;
  for (int i = 0; i < p.n; ++i)
    if (p.ops[i].code == TCK_S) l = i;
  return l;
}

template <int N, int REDLEN, int TG_>
struct CStreamCfg {
  static constexpr int D = 3, C = 4, NODES = N * N * N, NF = N * N, VOL = C * NODES;
  static constexpr int TG = TG_;
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  // metric buffer: the element's record (inv_jac | JxW | normals | face JxW)
  // | reduced-degree inv_jac
  static constexpr int M_IJ = CRec<N>::IJ;
  static constexpr int M_JW = CRec<N>::JW;
  static constexpr int M_FN = CRec<N>::FN;
  static constexpr int M_FJ = CRec<N>::FJ;
  static constexpr int M_RED = CRec<N>::LEN;
  static constexpr int MET = M_RED + ev(REDLEN);
  // layout: U x 2 | neighbour traces / face integrand | metric | 1/JxW | 4 work tiles
  static constexpr int OFF_U = 0;
  static constexpr int OFF_NB = 2 * ev(VOL);
  static constexpr int OFF_MET = OFF_NB + ev(6 * C * NF);
  static constexpr int OFF_IJW = OFF_MET + MET;
  static constexpr int WT = ev(VOL > 6 * C * NF ? VOL : 6 * C * NF);
  static constexpr int OFF_W = OFF_IJW + ev(NODES);
  static constexpr int OFF_IDS = OFF_W + 4 * WT;   // 3 slots x 8 ints
  static constexpr int OFF_MAT = OFF_IDS + 12;     // 3 slots x 4 doubles
  static constexpr int OFF_BAR = OFF_MAT + 12;     // U[0], U[1], metric
  static constexpr int OFF_Q = OFF_BAR + 4;
  static constexpr int TOTAL = OFF_Q + 2;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  static constexpr int RPL = (VOL + TG - 1) / TG;
};

namespace scurv {

// f(integral_constant<int, Q>) for every Q of the sequence (C++17 fold)
template <int... Q, typename F>
__device__ __forceinline__ void for_each_int(std::integer_sequence<int, Q...>, F&& f) {
  (f(std::integral_constant<int, Q>{}), ...);
}
template <int O, int... I>
__host__ __device__ constexpr std::integer_sequence<int, (I + O)...> offset_seq(
    std::integer_sequence<int, I...>) {
  return {};
}

// first point and stride of line l along direction m of an NN^3 grid
template <int NN>
__device__ __forceinline__ int lbase(int m, int l) {
  return m == 0 ? l * NN : (m == 1 ? (l % NN) + (l / NN) * NN * NN : l);
}
template <int NN>
__device__ __forceinline__ int lstride(int m) {
  return m == 0 ? 1 : (m == 1 ? NN : NN * NN);
}

// one line of a volume sweep (component c = item / n^2) along M with the
// n x n table at ctab[MOFF]; SUM3: the input is (in + in1 + in2) / JxW
template <int N, int M, int MOFF, bool SUM3>
__device__ __forceinline__ void vsweep_item(const CurvedStreamArgs& A, const double* in,
                                            double* out, int item, const double* in1 = nullptr,
                                            const double* in2 = nullptr,
                                            const double* ijw = nullptr) {
  constexpr int NODES = N * N * N, NN2 = N * N;
  constexpr int S = M == 0 ? 1 : (M == 1 ? N : NN2);
  const int c = item / NN2, l = item - c * NN2;
  const int lb = M == 0 ? l * N : (M == 1 ? (l % N) + (l / N) * NN2 : l);
  const int base = c * NODES + lb;
  double x[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    if constexpr (SUM3) {
      const int o = base + j * S;
      x[j] = (in[o] + in1[o] + in2[o]) * ijw[lb + j * S];
    } else {
      x[j] = in[base + j * S];
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(A.ctab[MOFF + i * N + j], x[j], s);
    out[base + i * S] = s;
  }
}

// one line of a 2-D sweep over the 6 x C face blocks (n x n each) along
// face direction M2 (0: fast index, 1: slow index)
template <int N, int M2, int MOFF>
__device__ __forceinline__ void fsweep_item(const CurvedStreamArgs& A, const double* in,
                                            double* out, int item) {
  constexpr int NF = N * N, S = M2 == 0 ? 1 : N;
  const int blk = item / N, l = item - blk * N;
  const int base = blk * NF + (M2 == 0 ? l * N : l);
  double x[N];
#pragma unroll
  for (int j = 0; j < N; ++j) x[j] = in[base + j * S];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s = fma(A.ctab[MOFF + i * N + j], x[j], s);
    out[base + i * S] = s;
  }
}

// y = T x with the n x n table at a compile-time offset of the kernel
// parameters (PLAN: the Taylor plan's blob, else ctab): constant-bank operands
template <int NN, int OFF, bool PLAN>
__device__ __forceinline__ void mat1d(const CurvedStreamArgs& A, const double (&x)[NN],
                                      double (&y)[NN]) {
#pragma unroll
  for (int i = 0; i < NN; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NN; ++j)
      s = fma(PLAN ? A.t.tab[OFF + i * NN + j] : A.ctab[OFF + i * NN + j], x[j], s);
    y[i] = s;
  }
}

// Curved S at NN = q+1 points (operator.py:286-306) as directional line
// tasks: out_v_c = ir sum_m G_mc d_m p, out_p = c2r sum_m sum_c G_mc d_m v_c,
// the direction-m share into tile p[m].  ij: (9, NN^3) metric of degree q.
template <int N, int NN, int TOFF, int TG>
__device__ __forceinline__ void curved_S_tasks(const CurvedStreamArgs& A, const double* cur,
                                               double* p0, double* p1, double* p2,
                                               const double* ij, double ir, double c2r, int tid) {
  constexpr int NODES = N * N * N, NN2 = NN * NN, NPQ = NN2 * NN;
  constexpr int PADT = ((3 * NN2 + 31) / 32) * 32;   // tasks per type, warp-aligned
  constexpr int NIT = (2 * PADT + TG - 1) / TG;
#pragma unroll 1
  for (int it = 0; it < NIT; ++it) {
    const int s = tid + it * TG;
    const int ty = s / PADT, r = s - ty * PADT;
    if (((2 * PADT) % TG == 0 || s < 2 * PADT) && r < 3 * NN2) {
      const int m = r / NN2, l = r - m * NN2;
      const int lb = lbase<NN>(m, l), S = lstride<NN>(m);
      double* out = (m == 0 ? p0 : (m == 1 ? p1 : p2)) + lb;
      if (ty == 0) {   // v_c = ir G_mc d_m p, c = 0..2
        double x[NN], g[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) x[j] = cur[3 * NODES + lb + j * S];
        mat1d<NN, TOFF, true>(A, x, g);
#pragma unroll
        for (int i = 0; i < NN; ++i) g[i] *= ir;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double* G = ij + (m * 3 + c) * NPQ + lb;
#pragma unroll
          for (int i = 0; i < NN; ++i) out[c * NODES + i * S] = G[i * S] * g[i];
        }
      } else {         // p = c2r sum_c G_mc d_m v_c
        double y[NN];
#pragma unroll
        for (int i = 0; i < NN; ++i) y[i] = 0.0;
#pragma unroll
        for (int c2 = 0; c2 < 3; ++c2) {
          double x[NN], g[NN];
#pragma unroll
          for (int j = 0; j < NN; ++j) x[j] = cur[c2 * NODES + lb + j * S];
          mat1d<NN, TOFF, true>(A, x, g);
          const double* G = ij + (m * 3 + c2) * NPQ + lb;
#pragma unroll
          for (int i = 0; i < NN; ++i) y[i] = fma(G[i * S], g[i], y[i]);
        }
#pragma unroll
        for (int i = 0; i < NN; ++i) out[3 * NODES + i * S] = c2r * y[i];
      }
    }
  }
  __syncthreads();
}

// t1 <- t1 + t2 + t3 on a degree-q field (element-wise ownership tid + j*TG,
// the accumulators' layout), optionally fused with the plan's accumulator op
template <int N, int NN, int TG, int RPL, int CODE, int WI>
__device__ __forceinline__ void sum3(const CurvedStreamArgs& A, double* t1, const double* t2,
                                     const double* t3, double (&acc)[RPL], int tid) {
  constexpr int NODES = N * N * N, NPQ = NN * NN * NN, ITEMS = 4 * NPQ;
  constexpr int NIT = (ITEMS + TG - 1) / TG;
#pragma unroll
  for (int j = 0; j < NIT; ++j) {
    const int f = tid + j * TG;
    if (ITEMS % TG == 0 || f < ITEMS) {
      const int qc = f / NPQ, pt = f - qc * NPQ;
      const int o = qc * NODES + pt;
      const double v = t1[o] + t2[o] + t3[o];
      t1[o] = v;
      if (CODE == TCK_ACC_SET) acc[j] = A.t.w[WI] * v;
      else if (CODE == TCK_ACC_ADD) acc[j] = acc[j] + A.t.w[WI] * v;
    }
  }
  __syncthreads();
}

// the plan, op by op; the four work tiles rotate: cur = tile(ci)
// projection / interpolation NF_ -> NT_ points in every direction
// (operator.py:308-325): in -> a -> b -> a, result in a.  SUM3: the input is
// the sum of the three partial tiles of an S op (its consumer).
template <int N, int TG, int NF_, int NT_, int TOFF, bool SUM3>
__device__ __forceinline__ void resize3(const CurvedStreamArgs& A, const double* in0,
                                        const double* in1, const double* in2, double* a,
                                        double* b, int tid) {
  constexpr int C = 4, NODES = N * N * N;
  constexpr int MX = NF_ > NT_ ? NF_ : NT_;
  constexpr int NIT = (C * MX * MX + TG - 1) / TG;
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    const int lo_ext = m == 0 ? 1 : (m == 1 ? NT_ : NT_ * NT_);
    const int hi_ext = m == 0 ? NF_ * NF_ : (m == 1 ? NF_ : 1);
    const int lines = lo_ext * hi_ext;
    const double* src0 = m == 0 ? in0 : (m == 1 ? a : b);
    double* dst0 = m == 1 ? b : a;
#pragma unroll 1
    for (int it = 0; it < NIT; ++it) {
      const int t = tid + it * TG;
      if (t < C * lines) {
        const int qc = t / lines, l = t - qc * lines;
        const int hi = l / lo_ext, lo = l - hi * lo_ext;
        const int so = qc * NODES + lo + hi * lo_ext * NF_;
        double x[NF_];
#pragma unroll
        for (int j = 0; j < NF_; ++j) {
          const int o = so + j * lo_ext;
          if (SUM3 && m == 0) x[j] = in0[o] + in1[o] + in2[o];
          else x[j] = src0[o];
        }
        double* dst = dst0 + qc * NODES + lo + hi * lo_ext * NT_;
#pragma unroll
        for (int i = 0; i < NT_; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < NF_; ++j) acc = fma(A.t.tab[TOFF + i * NF_ + j], x[j], acc);
          dst[i * lo_ext] = acc;
        }
      }
    }
    __syncthreads();
  }
}

// the plan, op by op; the four work tiles rotate: cur = tile(ci)
template <int N, int REDLEN, int STRIDE, bool SHIFT, int TG, int RPL, int I, typename IssueMet>
__device__ __forceinline__ void run_op(const CurvedStreamArgs& A, double* W0, int& ci,
                                       double (&acc)[N][RPL], const double* met, double ir,
                                       double c2r, int tid, IssueMet& issue_met) {
  using K = CStreamCfg<N, REDLEN, TG>;
  constexpr TckPlan P = sader::Plan<3, N, STRIDE, SHIFT>::P;
  constexpr TckStep op = P.ops[I];
  constexpr int PREV = P.ops[I > 0 ? I - 1 : 0].code;
  auto tile = [&](int i) { return W0 + ((ci + i) & 3) * K::WT; };
  if constexpr (op.code == TCK_S) {
    constexpr int q = op.a0 - 1;
    const double* ij = (q == N - 1) ? met + K::M_IJ : met + K::M_RED + red_off(P, N - 1, q);
    curved_S_tasks<N, op.a0, op.a1, TG>(A, tile(0), tile(1), tile(2), tile(3), ij, ir, c2r, tid);
    if constexpr (I == last_S(P)) issue_met();    // the metric buffer is free
    constexpr TckStep nx = P.ops[I + 1 < P.n ? I + 1 : I];
    constexpr bool fuse = I + 1 < P.n && (nx.code == TCK_ACC_SET || nx.code == TCK_ACC_ADD);
    if constexpr (I + 1 < P.n && nx.code == TCK_RESIZE) {
      // the resize sums the partials in its first sweep
    } else {
      constexpr int slot = fuse ? nx.a0 : 0;
      sum3<N, op.a0, TG, RPL, fuse ? nx.code : -1, I + 1>(A, tile(1), tile(2), tile(3),
                                                          acc[slot], tid);
      ci = (ci + 1) & 3;
    }
  } else if constexpr (op.code == TCK_RESIZE) {
    if constexpr (I > 0 && PREV == TCK_S) {
      // partials in tile(1..3); the S input tile(0) is free: result -> tile(0)
      resize3<N, TG, op.a0, op.a1, op.a2, true>(A, tile(1), tile(2), tile(3), tile(0), tile(1),
                                                tid);
    } else {
      resize3<N, TG, op.a0, op.a1, op.a2, false>(A, tile(0), nullptr, nullptr, tile(1), tile(2),
                                                 tid);
      ci = (ci + 1) & 3;
    }
  } else if constexpr (op.code == TCK_LOAD) {
    // cur <- acc (ownership layout).  No barrier before: the op before a LOAD
    // is an accumulator op reading cur at this thread's own indices, or a
    // resize / fused S accumulation that ended in a barrier.
    constexpr int NPQ = op.a1 * op.a1 * op.a1, ITEMS = 4 * NPQ;
    constexpr int NIT = (ITEMS + TG - 1) / TG;
    double* cur = tile(0);
#pragma unroll
    for (int j = 0; j < NIT; ++j) {
      const int f = tid + j * TG;
      if (ITEMS % TG == 0 || f < ITEMS) {
        const int qc = f / NPQ, pt = f - qc * NPQ;
        cur[qc * (N * N * N) + pt] = acc[op.a0][j];
      }
    }
    __syncthreads();
  } else {
    constexpr bool fused = I > 0 && PREV == TCK_S;
    if constexpr (!fused)
      sader::acc_op<3, N, TG, 1, op.a0, op.code, I>(A.t, acc[op.a0], tile(0), tid);
  }
}

template <int N, int REDLEN, int STRIDE, bool SHIFT, int TG, int RPL, typename IssueMet,
          int... I>
__device__ __forceinline__ void run_plan(const CurvedStreamArgs& A, double* W0, int& ci,
                                         double (&acc)[N][RPL], const double* met, double ir,
                                         double c2r, int tid, IssueMet& issue_met,
                                         std::integer_sequence<int, I...>) {
  (run_op<N, REDLEN, STRIDE, SHIFT, TG, RPL, I>(A, W0, ci, acc, met, ir, c2r, tid, issue_met),
   ...);
}

}  // namespace scurv

// KIND: 0..3 = operator output modes (OUT_MINVK, OUT_RHS, OUT_LSRK, OUT_ADERB);
// 8 = ADER kernel A (HDG), 9 = ADER kernel A (plain)
constexpr int kCurvedAderHdg = 8, kCurvedAder = 9;

template <int N, int KIND, int STRIDE, bool SHIFT>
struct CurvedKernelCfg {
  static constexpr bool ADER = KIND >= 8;
  static constexpr int REDLEN =
      ADER ? red_len(make_tck_plan(N - 1, STRIDE, SHIFT), N - 1) : 0;
#ifdef WK_CURVED_TG
  static constexpr int TG = N >= 6 ? WK_CURVED_TG : (N >= 4 ? 128 : 64);
#else
  static constexpr int TG = N >= 6 ? 256 : (N >= 4 ? 128 : 64);
#endif
  // CTAs per SM the register budget is sized for (shared memory allows 3 for
  // the operator at n = 6)
#ifdef WK_CURVED_MINB
  static constexpr int MINB = WK_CURVED_MINB;
#else
  static constexpr int MINB = 2;
#endif
  using K = CStreamCfg<N, REDLEN, TG>;
};

template <int N, int KIND, int STRIDE, bool SHIFT>
__global__ void __launch_bounds__(CurvedKernelCfg<N, KIND, STRIDE, SHIFT>::TG,
                                  CurvedKernelCfg<N, KIND, STRIDE, SHIFT>::MINB)
curved_stream_kernel(const __grid_constant__ CurvedStreamArgs A) {
  using KC = CurvedKernelCfg<N, KIND, STRIDE, SHIFT>;
  using K = typename KC::K;
  constexpr bool ADER = KC::ADER;
  constexpr bool HDG = KIND == kCurvedAderHdg;
  constexpr bool OPER = !ADER || HDG;        // the operator residual is evaluated
  constexpr int MODE = KIND;                 // operator output mode when !ADER
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, VOL = K::VOL, TG = K::TG;
  constexpr int RPL = K::RPL;
  constexpr int NN2 = N * N;
  constexpr int T_B = 0, T_BINV = NN2, T_DCO = 2 * NN2, T_DCOT = 3 * NN2;
  constexpr bool READ_RV = !ADER && (MODE == OUT_LSRK || MODE == OUT_ADERB);
  constexpr TckPlan PL = sader::Plan<3, N, STRIDE, SHIFT>::P;
  extern __shared__ __align__(128) double smem[];
  double* const nb = smem + K::OFF_NB;
  double* const met = smem + K::OFF_MET;
  double* const ijw = smem + K::OFF_IJW;
  double* const W0 = smem + K::OFF_W;
  double* const T0 = W0;
  double* const T1 = W0 + K::WT;
  double* const T2 = W0 + 2 * K::WT;
  double* const T3 = W0 + 3 * K::WT;
  int* const sids = reinterpret_cast<int*>(smem + K::OFF_IDS);
  double* const smat = smem + K::OFF_MAT;
  unsigned long long* const bar = reinterpret_cast<unsigned long long*>(smem + K::OFF_BAR);
  const int tid = threadIdx.x;
  WK_CHECK_SMEM(K::BYTES);
  const AffineArgs& op = A.t.op;
  const long long e_begin = op.e_begin;
  const long long ntiles = op.E;                  // one element per tile
  const double* const gU = op.u;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || op.a != 0.0);
  const double* const gsrc_r = (MODE == OUT_ADERB) ? op.v : op.r;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
  }

  // ---- copies ---------------------------------------------------------------
  // bulk copy (TMA) for pieces of an even number of doubles (16 B multiples,
  // 16 B aligned: every array base is a cudaMalloc pointer and the element
  // offset is a multiple of the piece), else cp.async by all threads; the
  // piece sizes are compile-time, so only one path is emitted per piece
  auto issue_pieces = [&](auto&& pieces, unsigned long long* b) {
    if (tid == 0) {
      unsigned tx = 0;
      pieces([&](double*, const double*, int n) {
        if ((n & 1) == 0) tx += (unsigned)n * 8u;
      });
      mbar_arrive_expect_tx(b, tx);
      pieces([&](double* dst, const double* src, int n) {
        if ((n & 1) == 0) bulk_g2s(dst, src, (unsigned)n * 8u, b);
      });
    }
    pieces([&](double* dst, const double* src, int n) {
      if (n & 1)
        for (int j = tid; j < n; j += TG) cp_async8(dst + j, src + j);
    });
  };
  // the metric buffer's per-element contiguous pieces: f(dst, src, n_doubles)
  auto met_pieces = [&](long long e, auto&& f) {
    // the operator reads the whole record, the plain Taylor loop its inv_jac
    if (OPER) f(met, A.rec + e * CRec<N>::LEN, CRec<N>::LEN);
    else f(met, A.rec + e * CRec<N>::LEN, CRec<N>::JW);
    if constexpr (ADER) {
      // reduced-degree metrics the plan's S ops read (compile-time degree list)
      scurv::for_each_int(std::make_integer_sequence<int, N - 1>{}, [&](auto qc) {
        constexpr int q = decltype(qc)::value;
        using PP = sader::Plan<3, N, STRIDE, SHIFT>;
        if constexpr (plan_uses_S(PP::P, q)) {
          constexpr int npq = 9 * (q + 1) * (q + 1) * (q + 1);
          f(met + K::M_RED + red_off(PP::P, N - 1, q), A.inv_jac[q] + e * npq, npq);
        }
      });
    }
  };
  auto issue_u = [&](long long t, int b) {
    const long long e = e_begin + t;
    issue_pieces([&](auto&& f) { f(smem + K::OFF_U + b * K::ev(VOL), gU + e * VOL, VOL); },
                 &bar[b]);
  };
  auto issue_met_t = [&](long long t) {
    const long long e = e_begin + t;
    issue_pieces([&](auto&& f) { met_pieces(e, f); }, &bar[2]);
  };
  auto issue_nb = [&](long long t, const int* ids) {
    if (!OPER) return;
    (void)t;
    // neighbour face-node values [f][c][fn] (GL), all components
    for (int t2 = tid; t2 < 6 * C * NF; t2 += TG) {
      const int f = t2 / (C * NF), rest = t2 - f * (C * NF);
      const int c = rest / NF, fn = rest - c * NF;
      const int nbe = ids[f];
      WK_CHECK_NBR(op, nbe);
      if (nbe >= 0) {
        cp_async8(nb + t2, gU + ((long long)nbe * C + c) * NODES + face_to_node<N>(f >> 1, 1 - (f & 1), fn));
      } else if (op.has_ghost && nbe <= -2) {
        cp_async8(nb + t2, op.ghost + ((long long)ghost_slot(nbe) * C + c) * NF + fn);
      }
    }
  };

  // ---- tile queue (see affine_stream_kernel) + id / material rings --------
  long long* const qslot = reinterpret_cast<long long*>(smem + K::OFF_Q);
  const long long kNone = ntiles;
  const long long dyn0 = 2LL * gridDim.x;
  const unsigned qcap = (unsigned)(ntiles + 4LL * gridDim.x + 64);
  long long tile = blockIdx.x;   // grid <= ntiles (launcher)
  long long nxt = tile + gridDim.x < ntiles ? tile + gridDim.x : kNone;
  unsigned raw = 0;
  bool pend = false;
  auto load_meta = [&](long long t, int slot) {    // synchronous (prologue only)
    if (tid < 6) sids[slot * 8 + tid] = t < ntiles ? __ldg(op.nbr + (e_begin + t) * 6 + tid) : -1;
    else if (tid >= 8 && tid < 12)
      smat[slot * 4 + tid - 8] = t < ntiles ? __ldg(op.mat + (e_begin + t) * kMatStride + tid - 8) : 0.0;
  };
  load_meta(tile, 0);
  load_meta(nxt, 1);
  if (tid == 0) {
    long long w = kNone;
    if (nxt < ntiles) {
      w = dyn0 + (long long)atomic_claim(op.sched, qcap);
      if (w >= ntiles) w = kNone;
    }
    qslot[1] = w;
    pend = w < ntiles;
    if (pend) raw = atomic_claim(op.sched, qcap);
  }
  __syncthreads();
  long long nn = qslot[1];
  issue_u(tile, 0);
  issue_met_t(tile);
  issue_nb(tile, sids);
  cp_async_commit();
  int buf = 0;
  unsigned it = 0;
  while (tile < ntiles) {
    const int sl_cur = it % 3, sl_nxt = (it + 1) % 3, sl_nn = (it + 2) % 3;
    if (nxt < ntiles) issue_u(nxt, buf ^ 1);
    if (op.l2pf && tid == 0 && nn < ntiles) {
      bulk_prefetch_l2(gU + (e_begin + nn) * VOL, (unsigned)(VOL * 8) & ~15u);
      bulk_prefetch_l2(A.rec + (e_begin + nn) * CRec<N>::LEN,
                       (unsigned)((OPER ? CRec<N>::LEN : CRec<N>::JW) * 8) & ~15u);
    }
    if (tid == 0) {
      long long w = kNone;
      if (pend) {
        w = dyn0 + (long long)raw;
        if (w >= ntiles) w = kNone;
      }
      qslot[it & 1] = w;
      pend = w < ntiles;
      if (pend) raw = atomic_claim(op.sched, qcap);
    }
    const long long e = e_begin + tile;
    const long long goff = e * VOL;
    double rv[RPL];
    if (READ_RV) {
      if (read_r) {
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          const int idx = tid + j * TG;
          rv[j] = (idx < VOL) ? __ldcs(gsrc_r + goff + idx) : 0.0;
        }
      }
    }
    mbar_wait(&bar[buf], (it >> 1) & 1u);
    mbar_wait(&bar[2], it & 1u);
    cp_async_wait<0>();
    __syncthreads();
    const long long nnn = qslot[it & 1];
    // ids / material of tile nn into their ring slot by cp.async (its last
    // readers were in the previous iteration): committed with this
    // iteration's neighbour-trace group, complete at the next iteration's
    // wait, read when nn is the next tile (ids, issue_nb) and the current one
    // (material).  A register load here exposed its full latency to warp 0,
    // and the CTA waited for warp 0 at the next barrier (8 % of kernel B).
    if (nn < ntiles) {
      if (tid < 6) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(sids + sl_nn * 8 + tid)),
                     "l"(op.nbr + (e_begin + nn) * 6 + tid));
      } else if (tid >= 8 && tid < 12) {
        cp_async8(smat + sl_nn * 4 + tid - 8, op.mat + (e_begin + nn) * kMatStride + tid - 8);
      }
    }

    const double* const us = smem + K::OFF_U + buf * K::ev(VOL);
    const int* const ids = sids + sl_cur * 8;
    const double ir = smat[sl_cur * 4 + 0], c2r = smat[sl_cur * 4 + 1];
    const double tau = smat[sl_cur * 4 + 2], irt = smat[sl_cur * 4 + 3];
    bool met_issued = false;
    auto issue_met_next = [&]() {
      if (!met_issued) {
        met_issued = true;
        if (nxt < ntiles) issue_met_t(nxt);
        cp_async_commit();
      }
    };

    // ---- P1: Gauss values Q = B (x)3 U -> T0; neighbour traces B (x)2 in nb
    {
#ifndef WK_CURVED_FPAIR
#define WK_CURVED_FPAIR 1
#endif
      // face lines two per thread (independent blocks f and f + FH) when that
      // brings the volume + face lines of a sweep within one pass of the CTA
      // (n = 6: 144 + 144 lines -> 144 + 72 for 256 threads)
      constexpr int VI = 4 * NN2, FI = OPER ? 6 * C * N : 0;
      constexpr bool PAIR = WK_CURVED_FPAIR && VI + FI > TG && VI + FI / 2 <= TG;
      constexpr int FH = PAIR ? FI / 2 : FI;
      constexpr int NIT = (VI + FH + TG - 1) / TG;
#pragma unroll 1
      for (int i = 0; i < NIT; ++i) {
        const int t = tid + i * TG;
        if (t < VI) {
          scurv::vsweep_item<N, 0, T_B, false>(A, us, T1, t);
        } else if (OPER && t < VI + FH) {
          scurv::fsweep_item<N, 0, T_B>(A, nb, T3, t - VI);
          if (PAIR) scurv::fsweep_item<N, 0, T_B>(A, nb, T3, t - VI + FH);
        }
      }
      __syncthreads();
#pragma unroll 1
      for (int i = 0; i < NIT; ++i) {
        const int t = tid + i * TG;
        if (t < VI) {
          scurv::vsweep_item<N, 1, T_B, false>(A, T1, T2, t);
        } else if (OPER && t < VI + FH) {
          scurv::fsweep_item<N, 1, T_B>(A, T3, nb, t - VI);
          if (PAIR) scurv::fsweep_item<N, 1, T_B>(A, T3, nb, t - VI + FH);
        }
      }
      __syncthreads();
      constexpr int NIT2 = (VI + TG - 1) / TG;
#pragma unroll
      for (int i = 0; i < NIT2; ++i) {
        const int t = tid + i * TG;
        if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 2, T_B, false>(A, T2, T0, t);
      }
      __syncthreads();
    }
    const double* const Q = T0;
    if constexpr (OPER) {
      // ---- P2: face integrand u_hat - F_n(own)/2 (operator.py:217-239) at the
      //      face Gauss points, in place over the neighbour traces; own traces
      //      from Q by the endpoint rows of B^{-1}; 1/JxW
      for (int t2 = tid; t2 < 6 * NF; t2 += TG) {
        const int f = t2 / NF, fn = t2 - f * NF;
        const int m = f >> 1, side = f & 1;
        const int lb = scurv::lbase<N>(m, fn), S = scurv::lstride<N>(m);
        double own[C], oth[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j)
            s = fma(side ? A.ctab[T_BINV + (N - 1) * N + j] : A.ctab[T_BINV + j],
                    Q[c * NODES + lb + j * S], s);
          own[c] = s;
        }
        const int nbr = ids[f];
        if (nbr == -1) {
#pragma unroll
          for (int c = 0; c < 3; ++c) oth[c] = own[c];
          oth[3] = -own[3];
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) oth[c] = nb[(f * C + c) * NF + fn];
        }
        const double* nrm_p = met + K::M_FN + f * 3 * NF + fn;
        double nrm[3], vn_o = 0.0, vn_x = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          nrm[i] = nrm_p[i * NF];
          vn_o = fma(nrm[i], own[i], vn_o);
          vn_x = fma(nrm[i], oth[i], vn_x);
        }
        double pv = 0.5 * ir * oth[3];
        double pp = 0.5 * c2r * vn_x;
        if (op.stab) {
          pv += 0.5 * irt * (vn_o - vn_x);
          pp += 0.5 * c2r * tau * (own[3] - oth[3]);
        }
        const double fj = met[K::M_FJ + f * NF + fn];
#pragma unroll
        for (int i = 0; i < 3; ++i) nb[(f * C + i) * NF + fn] = pv * nrm[i] * fj;
        nb[(f * C + 3) * NF + fn] = pp * fj;
      }
      for (int pt = tid; pt < NODES; pt += TG) ijw[pt] = 1.0 / met[K::M_JW + pt];
      __syncthreads();
      // ---- P3: directional line tasks -> partial residuals T1, T2, T3 -------
      //   two balanced task types per (direction m, line l):
      //   'v': D p once, then the three velocity outputs (strong + weak + lifts)
      //   'p': D v_0..2, then the pressure output       (~n^2 (2d+... ) FMAs each)
      {
        constexpr int PADT = ((3 * NN2 + 31) / 32) * 32;   // tasks per type, warp-aligned
        constexpr int NIT = (2 * PADT + TG - 1) / TG;
#pragma unroll 1
        for (int i = 0; i < NIT; ++i) {
          const int s = tid + i * TG;
          const int ty = s / PADT, r = s - ty * PADT;
          if (((2 * PADT) % TG == 0 || s < 2 * PADT) && r < 3 * NN2) {
            const int m = r / NN2, l = r - m * NN2;
            const int lb = scurv::lbase<N>(m, l), S = scurv::lstride<N>(m);
            const double* jwl = met + K::M_JW + lb;
            double* const outm = (m == 0 ? T1 : (m == 1 ? T2 : T3)) + lb;
            // out[i] = ya[i] + (D_co^T wa)[i] + the face lifts at both line ends
            auto finish = [&](const double (&ya)[N], const double (&wa)[N], int c) {
              const double f0 = nb[((2 * m) * C + c) * NF + l];
              const double f1 = nb[((2 * m + 1) * C + c) * NF + l];
              double* out = outm + c * NODES;
#pragma unroll
              for (int i2 = 0; i2 < N; ++i2) {
                double v = ya[i2];
#pragma unroll
                for (int j = 0; j < N; ++j) v = fma(A.ctab[T_DCOT + i2 * N + j], wa[j], v);
                out[i2 * S] = fma(A.ctab[T_BINV + i2], f0,
                                  fma(A.ctab[T_BINV + (N - 1) * N + i2], f1, v));
              }
            };
            if (ty == 0) {
              double pl[N], gp[N];
#pragma unroll
              for (int j = 0; j < N; ++j) pl[j] = Q[3 * NODES + lb + j * S];
              scurv::mat1d<N, T_DCO, false>(A, pl, gp);
              const double hv = 0.5 * ir;
#pragma unroll
              for (int j = 0; j < N; ++j) {      // fold 1/2 ir JxW into p and D p
                const double h = hv * jwl[j * S];
                pl[j] *= -h;
                gp[j] *= h;
              }
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                const double* G = met + K::M_IJ + (m * 3 + c) * NODES + lb;
                double ya[N], wa[N];
#pragma unroll
                for (int j = 0; j < N; ++j) {
                  const double g = G[j * S];
                  ya[j] = g * gp[j];     // strong: 1/2 JxW ir G_mc d_m p
                  wa[j] = g * pl[j];     // weak flux: -1/2 JxW ir G_mc p
                }
                finish(ya, wa, c);
              }
            } else {
              double ya[N], wa[N];
#pragma unroll
              for (int j = 0; j < N; ++j) ya[j] = wa[j] = 0.0;
#pragma unroll
              for (int c2 = 0; c2 < 3; ++c2) {
                double x[N], g[N];
#pragma unroll
                for (int j = 0; j < N; ++j) x[j] = Q[c2 * NODES + lb + j * S];
                scurv::mat1d<N, T_DCO, false>(A, x, g);
                const double* G = met + K::M_IJ + (m * 3 + c2) * NODES + lb;
#pragma unroll
                for (int j = 0; j < N; ++j) {
                  const double gm = G[j * S];
                  ya[j] = fma(gm, g[j], ya[j]);
                  wa[j] = fma(gm, x[j], wa[j]);
                }
              }
              const double hp = 0.5 * c2r;
#pragma unroll
              for (int j = 0; j < N; ++j) {
                const double h = hp * jwl[j * S];
                ya[j] = h * ya[j];
                wa[j] = -h * wa[j];
              }
              finish(ya, wa, 3);
            }
          }
        }
        __syncthreads();
      }
      // the neighbour traces are consumed: fetch the next element's
      if (nxt < ntiles) issue_nb(nxt, sids + sl_nxt * 8);
      if constexpr (!ADER) issue_met_next();      // metric consumed too
      else cp_async_commit();
      if constexpr (!ADER) {
        // ---- P4: W (GL) = B^{-1} (x)3 [(R_0 + R_1 + R_2) / JxW] -> T0 ------
        constexpr int VI = 4 * NN2;
        constexpr int NIT = (VI + TG - 1) / TG;
#pragma unroll
        for (int i = 0; i < NIT; ++i) {
          const int t = tid + i * TG;
          if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 0, T_BINV, true>(A, T1, T0, t, T2, T3, ijw);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NIT; ++i) {
          const int t = tid + i * TG;
          if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 1, T_BINV, false>(A, T0, T1, t);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NIT; ++i) {
          const int t = tid + i * TG;
          if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 2, T_BINV, false>(A, T1, T0, t);
        }
        __syncthreads();
        // ---- operator outputs (coalesced) -----------------------------------
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          const int idx = tid + j * TG;
          if (idx < VOL) {
            const double v = T0[idx];
            if (MODE == OUT_MINVK) {
              op.out[goff + idx] = v;
            } else if (MODE == OUT_RHS) {
              op.out[goff + idx] = -v;
            } else if (MODE == OUT_LSRK) {
              const double f = -v * op.dt;
              const double rr = read_r ? fma(op.a, rv[j], f) : f;
              if (!op.r_dead) op.r[goff + idx] = rr;
              op.u_out[goff + idx] = fma(op.b, rr, us[idx]);
            } else if (MODE == OUT_ADERB) {
              op.out[goff + idx] = rv[j] - v;
            }
          }
        }
      }
    }
    if constexpr (ADER) {
      double acc[N][RPL];
      int ci;
      if constexpr (HDG) {
        // W_q = (R_0 + R_1 + R_2) / JxW -> T1, fused with the plan's ACC_SET
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          const int idx = tid + j * TG;
          if (VOL % TG == 0 || idx < VOL) {
            const int pt = idx % NODES;
            const double v = (T1[idx] + T2[idx] + T3[idx]) * ijw[pt];
            T1[idx] = v;
            acc[N - 1][j] = A.t.w[0] * v;
          }
        }
        __syncthreads();
        // V = U - dt B^{-1} (x)3 W_q
        constexpr int VI = 4 * NN2;
        constexpr int NIT = (VI + TG - 1) / TG;
#pragma unroll
        for (int i = 0; i < NIT; ++i) {
          const int t = tid + i * TG;
          if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 0, T_BINV, false>(A, T1, T0, t);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NIT; ++i) {
          const int t = tid + i * TG;
          if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 1, T_BINV, false>(A, T0, T2, t);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < NIT; ++i) {
          const int t = tid + i * TG;
          if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 2, T_BINV, false>(A, T2, T0, t);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          const int idx = tid + j * TG;
          if (idx < VOL) A.t.v_out[goff + idx] = us[idx] - A.t.dt * T0[idx];
        }
        __syncthreads();
        ci = 1;
      } else {
        sader::acc_op<3, N, TG, 1, N - 1, TCK_ACC_SET, 0>(A.t, acc[N - 1], T0, tid);
        ci = 0;
      }
      // ---- Taylor loop at the Gauss points, compile-time plan (op 0 done) ----
      scurv::run_plan<N, KC::REDLEN, STRIDE, SHIFT, TG, RPL>(
          A, W0, ci, acc, met, ir, c2r, tid, issue_met_next,
          scurv::offset_seq<1>(std::make_integer_sequence<int, PL.n - 1>{}));
      issue_met_next();      // (a plan without S)
      // y = B^{-1} acc_k
      double* cur = W0 + (ci & 3) * K::WT;
      double* t1 = W0 + ((ci + 1) & 3) * K::WT;
      double* t2 = W0 + ((ci + 2) & 3) * K::WT;
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        const int idx = tid + j * TG;
        if (VOL % TG == 0 || idx < VOL) cur[idx] = acc[N - 1][j];
      }
      __syncthreads();
      constexpr int VI = 4 * NN2;
      constexpr int NIT = (VI + TG - 1) / TG;
#pragma unroll
      for (int i = 0; i < NIT; ++i) {
        const int t = tid + i * TG;
        if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 0, T_BINV, false>(A, cur, t1, t);
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < NIT; ++i) {
        const int t = tid + i * TG;
        if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 1, T_BINV, false>(A, t1, t2, t);
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < NIT; ++i) {
        const int t = tid + i * TG;
        if (VI % TG == 0 || t < VI) scurv::vsweep_item<N, 2, T_BINV, false>(A, t2, t1, t);
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        const int idx = tid + j * TG;
        if (idx < VOL) A.t.y[goff + idx] = t1[idx];
      }
    }
    __syncthreads();   // free the work tiles and the U stage
    buf ^= 1;
    ++it;
    tile = nxt;
    nxt = nn;
    nn = nnn;
  }
  sched_done(op.sched, tid == 0, pend, raw);
}

}  // namespace wk
