// Persistent, TMA-streamed kernels for curved (per-point metric) 3-D cells:
// the fused operator (LSRK stage, rhs, M^{-1}K, ADER kernel B) and ADER
// kernel A with the compile-time Taylor plan (wk_stream_ader.cuh).
//
// Arithmetic: curved_residual (wk_curved.cuh) — the reference's quadrature
// split form (operator.py:149-246) with the GeometryCache arrays
// (mesh.py:162-188), fused with the inverse mass, M^{-1}K = B^{-1}(x)3 [R/JxW]
// (operator.py:250-258) — restructured for streaming:
//   * one element per tile, persistent CTAs claiming tiles from the ordered
//     tile queue; everything the element needs that is contiguous per element
//     (U, the inverse Jacobian and JxW at the Gauss points, face normals and
//     face JxW, and for kernel A the metric at the reduced TCK degrees) is
//     streamed into the next stage by cp.async.bulk while the current element
//     is computed; the neighbours' face-node values by cp.async;
//   * the 1-D tables B, B^{-1}, D_co (and the plan's matrices) are kernel
//     parameters (constant bank), sweeps have compile-time extents;
//   * three work tiles: Gauss values, scratch (own face traces, then one
//     weak-flux direction at a time) and the residual; the face integrand
//     overwrites the neighbour traces in the stage, so the whole kernel fits
//     two CTAs per SM at n = 6 (config 3).
#pragma once
#include "wk_curved.cuh"
#include "wk_stream_ader.cuh"

namespace wk {

constexpr int kCTab = 5 * kMaxN * kMaxN;

struct CurvedStreamArgs {
  TckStreamArgs t;                 // t.op: operator inputs / outputs, tile queue; t.w, t.tab: plan
  const double* inv_jac[kMaxN];    // [q]: (E, d, d, (q+1)^d) at the degree-q Gauss points
  const double* jxw;               // (E, n^d) at the degree-k Gauss points
  const double* fnormal[6];        // (E, d, n^{d-1}) per face 2m+s
  const double* fjxw[6];           // (E, n^{d-1})
  double ctab[kCTab];              // B | B^{-1} | D_co | D_co^T | B^T, n x n each
};

__host__ __device__ constexpr bool stream_curved_supported(int D, int N) {
  return D == 3 && N >= 2 && N <= 7;   // n = 8 tiles exceed shared memory (two stages)
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

template <int N, int REDLEN>
struct CStreamCfg {
  static constexpr int D = 3, C = 4, NODES = N * N * N, NF = N * N, VOL = C * NODES;
  static constexpr int TG0 = ((NODES + 31) / 32) * 32;
  static constexpr int TG = TG0 < 64 ? 64 : (TG0 > 256 ? 256 : TG0);
  static constexpr int ev(int x) { return (x + 1) / 2 * 2; }
  // stage: U | inv_jac | JxW | normals | face JxW | neighbour traces | reduced metrics
  static constexpr int S_U = 0;
  static constexpr int S_IJ = S_U + ev(VOL);
  static constexpr int S_JW = S_IJ + ev(9 * NODES);
  static constexpr int S_FN = S_JW + ev(NODES);
  static constexpr int S_FJ = S_FN + ev(6 * 3 * NF);
  static constexpr int S_NB = S_FJ + ev(6 * NF);
  static constexpr int S_RED = S_NB + ev(6 * C * NF);
  static constexpr int STAGE = S_RED + ev(REDLEN);
  // work tiles (also hold the 6 x C x n^2 face-trace sets: larger than a
  // volume tile for n < 6)
  static constexpr int WT = ev(VOL > 6 * C * NF ? VOL : 6 * C * NF);
  static constexpr int W_A = 2 * STAGE;
  static constexpr int W_B = W_A + WT;
  static constexpr int W_R = W_B + WT;
  static constexpr int OFF_IDS = W_R + WT;        // 3 slots x 8 ints
  static constexpr int OFF_MAT = OFF_IDS + 12;    // 3 slots x 4 doubles
  static constexpr int OFF_BAR = OFF_MAT + 12;
  static constexpr int OFF_Q = OFF_BAR + 2;
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

// sweep of NBLK contiguous tensors (DIRS directions of N points) along M
// with the n x n table at ctab[MOFF] (constant bank)
template <int N, int DIRS, int M, int NBLK, int TG, int MOFF>
__device__ __forceinline__ void tsweep(const CurvedStreamArgs& A, const double* in, double* out,
                                       int tid) {
  constexpr int SM = M == 0 ? 1 : (M == 1 ? N : N * N);
  constexpr int PER = DIRS == 3 ? N * N * N : (DIRS == 2 ? N * N : N);
  constexpr int LINES = PER / N;
  constexpr int ITEMS = NBLK * LINES;
  constexpr int NIT = (ITEMS + TG - 1) / TG;
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int t = tid + it * TG;
    if (ITEMS % TG == 0 || t < ITEMS) {
      const int blk = t / LINES, l = t - (t / LINES) * LINES;
      const int lo = l % SM, hi = l / SM;
      const int base = blk * PER + lo + hi * SM * N;
      double x[N];
#pragma unroll
      for (int j = 0; j < N; ++j) x[j] = in[base + j * SM];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) s = fma(A.ctab[MOFF + i * N + j], x[j], s);
        out[base + i * SM] = s;
      }
    }
  }
}

// all three directions of a volume tile (4 components): a -> b -> c -> b;
// returns the buffer holding the result
template <int N, int TG, int MOFF>
__device__ __forceinline__ double* vsweep3(const CurvedStreamArgs& A, const double* src,
                                           double* b1, double* b2, int tid) {
  tsweep<N, 3, 0, 4, TG, MOFF>(A, src, b1, tid);
  __syncthreads();
  tsweep<N, 3, 1, 4, TG, MOFF>(A, b1, b2, tid);
  __syncthreads();
  tsweep<N, 3, 2, 4, TG, MOFF>(A, b2, b1, tid);
  __syncthreads();
  return b1;
}

// curved S at NN = q+1 points (operator.py:286-306) with the staged metric
// of degree q: out_v = ir G^T grad p, out_p = c2r sum_{m,i} G_mi d_m v_i
template <int N, int NN, int TOFF, int TG>
__device__ __forceinline__ void curved_S(const CurvedStreamArgs& A, const double* cur, double* nxt,
                                         const double* ij, double ir, double c2r, int tid) {
  constexpr int NODES = N * N * N, C = 4;
  constexpr int NPT = NN * NN * NN;
  constexpr int NIT = (NPT + TG - 1) / TG;
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int pt = tid + it * TG;
    if (NPT % TG == 0 || pt < NPT) {
      double grad[3][C];
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int sm_ = m == 0 ? 1 : (m == 1 ? NN : NN * NN);
        const int im = (pt / sm_) % NN;
        const int base = pt - im * sm_;
        double row[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) row[j] = A.t.tab[TOFF + im * NN + j];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < NN; ++j) s = fma(row[j], cur[c * NODES + base + j * sm_], s);
          grad[m][c] = s;
        }
      }
      double sv[3] = {0.0, 0.0, 0.0}, sp = 0.0;
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double gmi = ij[(m * 3 + i) * NPT + pt];
          sv[i] = fma(gmi, grad[m][3], sv[i]);
          sp = fma(gmi, grad[m][i], sp);
        }
#pragma unroll
      for (int i = 0; i < 3; ++i) nxt[i * NODES + pt] = ir * sv[i];
      nxt[3 * NODES + pt] = c2r * sp;
    }
  }
  __syncthreads();
}

template <int N, int REDLEN, int STRIDE, bool SHIFT, int I, int RPL>
__device__ __forceinline__ void run_op(const CurvedStreamArgs& A, double*& cur, double*& nxt,
                                       double (&acc)[N][RPL], const double* stage,
                                       double ir, double c2r, int tid) {
  using K = CStreamCfg<N, REDLEN>;
  constexpr TckPlan P = sader::Plan<3, N, STRIDE, SHIFT>::P;
  constexpr TckStep op = P.ops[I];
  if constexpr (op.code == TCK_S) {
    constexpr int q = op.a0 - 1;
    const double* ij = (q == N - 1) ? stage + K::S_IJ : stage + K::S_RED + red_off(P, N - 1, q);
    curved_S<N, op.a0, op.a1, K::TG>(A, cur, nxt, ij, ir, c2r, tid);
    double* tt = cur;
    cur = nxt;
    nxt = tt;
  } else if constexpr (op.code == TCK_RESIZE) {
    sader::resize<3, N, K::TG, 1, op.a0, op.a1, op.a2>(A.t, cur, nxt, tid);
  } else {
    sader::acc_op<3, N, K::TG, 1, op.a0, op.code, I>(A.t, acc[op.a0], cur, tid);
  }
}

template <int N, int REDLEN, int STRIDE, bool SHIFT, int RPL, int... I>
__device__ __forceinline__ void run_plan(const CurvedStreamArgs& A, double*& cur, double*& nxt,
                                         double (&acc)[N][RPL], const double* stage, double ir,
                                         double c2r, int tid, std::integer_sequence<int, I...>) {
  (run_op<N, REDLEN, STRIDE, SHIFT, I, RPL>(A, cur, nxt, acc, stage, ir, c2r, tid), ...);
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
  using K = CStreamCfg<N, REDLEN>;
};

template <int N, int KIND, int STRIDE, bool SHIFT>
__global__ void __launch_bounds__(CurvedKernelCfg<N, KIND, STRIDE, SHIFT>::K::TG)
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
  extern __shared__ __align__(128) double smem[];
  double* const wA = smem + K::W_A;
  double* const wB = smem + K::W_B;
  double* const wR = smem + K::W_R;
  int* const sids = reinterpret_cast<int*>(smem + K::OFF_IDS);
  double* const smat = smem + K::OFF_MAT;
  unsigned long long* const bar = reinterpret_cast<unsigned long long*>(smem + K::OFF_BAR);
  const int tid = threadIdx.x;
  const AffineArgs& op = A.t.op;
  const long long e_begin = op.e_begin;
  const long long ntiles = op.E;                  // one element per tile
  const double* const gU = op.u;
  const bool read_r = READ_RV && (MODE == OUT_ADERB || op.a != 0.0);
  const double* const gsrc_r = (MODE == OUT_ADERB) ? op.v : op.r;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }

  // reduced-degree metrics the plan's S ops read (compile-time degree list)
  auto red_piece = [&](auto qc, long long e, double* st, auto&& f) {
    if constexpr (ADER) {
      constexpr int q = decltype(qc)::value;
      constexpr TckPlan P = sader::Plan<3, N, STRIDE, SHIFT>::P;
      if constexpr (plan_uses_S(P, q)) {
        constexpr int npq = 9 * (q + 1) * (q + 1) * (q + 1);
        f(st + K::S_RED + red_off(P, N - 1, q), A.inv_jac[q] + e * npq, npq);
      }
    }
  };
  auto red_pieces = [&](long long e, double* st, auto&& f, auto seq) {
    scurv::for_each_int(seq, [&](auto qc) { red_piece(qc, e, st, f); });
  };
  // the per-element contiguous arrays of tile t: f(dst, src, n_doubles)
  auto each_piece = [&](long long e, double* st, auto&& f) {
    f(st + K::S_U, gU + e * VOL, VOL);
    if (OPER || ADER) f(st + K::S_IJ, A.inv_jac[N - 1] + e * 9 * NODES, 9 * NODES);
    if (OPER) {
      f(st + K::S_JW, A.jxw + e * NODES, NODES);
#pragma unroll
      for (int fc = 0; fc < 6; ++fc) {
        f(st + K::S_FN + fc * 3 * NF, A.fnormal[fc] + e * 3 * NF, 3 * NF);
        f(st + K::S_FJ + fc * NF, A.fjxw[fc] + e * NF, NF);
      }
    }
    if constexpr (ADER) {
      red_pieces(e, st, f, std::make_integer_sequence<int, N - 1>{});
    }
  };
  // bulk copy (TMA) when 16-byte sized and aligned, else cp.async by all threads
  auto bulk_ok = [](const double* src, int n) {
    return ((n * 8) & 15) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0);
  };
  auto issue = [&](long long t, int b, const int* ids) {
    const long long e = e_begin + t;
    double* st = smem + b * K::STAGE;
    unsigned tx = 0;
    each_piece(e, st, [&](double*, const double* src, int n) {
      if (bulk_ok(src, n)) tx += (unsigned)n * 8u;
    });
    if (tid == 0) mbar_arrive_expect_tx(&bar[b], tx);
    each_piece(e, st, [&](double* dst, const double* src, int n) {
      if (bulk_ok(src, n)) {
        if (tid == 0) bulk_g2s(dst, src, (unsigned)n * 8u, &bar[b]);
      } else {
        for (int j = tid; j < n; j += TG) cp_async8(dst + j, src + j);
      }
    });
    if (OPER) {
      // neighbour face-node values [f][c][fn] (GL), all components
      for (int t2 = tid; t2 < 6 * C * NF; t2 += TG) {
        const int f = t2 / (C * NF), rest = t2 - f * (C * NF);
        const int c = rest / NF, fn = rest - c * NF;
        const int nb = ids[f];
        if (nb >= 0) {
          cp_async8(st + K::S_NB + t2,
                    gU + ((long long)nb * C + c) * NODES + face_to_node<N>(f >> 1, 1 - (f & 1), fn));
        } else if (op.has_ghost && nb <= -2) {
          cp_async8(st + K::S_NB + t2, op.ghost + ((long long)ghost_slot(nb) * C + c) * NF + fn);
        }
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
  issue(tile, 0, sids);
  cp_async_commit();
  int buf = 0;
  unsigned it = 0;
  while (tile < ntiles) {
    const int sl_cur = it % 3, sl_nxt = (it + 1) % 3, sl_nn = (it + 2) % 3;
    if (nxt < ntiles) issue(nxt, buf ^ 1, sids + sl_nxt * 8);
    cp_async_commit();
    // ids / material of tile nn (published at the end of this iteration)
    int idr = -1;
    double matr = 0.0;
    if (tid < 6 && nn < ntiles) idr = __ldg(op.nbr + (e_begin + nn) * 6 + tid);
    if (tid >= 8 && tid < 12 && nn < ntiles) matr = __ldg(op.mat + (e_begin + nn) * kMatStride + tid - 8);
    if (op.l2pf && tid == 0 && nn < ntiles) {
      bulk_prefetch_l2(gU + (e_begin + nn) * VOL, (unsigned)(VOL * 8) & ~15u);
      bulk_prefetch_l2(A.inv_jac[N - 1] + (e_begin + nn) * 9 * NODES, (unsigned)(9 * NODES * 8) & ~15u);
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
    cp_async_wait<1>();
    __syncthreads();
    const long long nnn = qslot[it & 1];

    double* const st = smem + buf * K::STAGE;
    const double* const us = st + K::S_U;
    const double* const ij = st + K::S_IJ;
    const double* const jw = st + K::S_JW;
    double* const nbt = st + K::S_NB;
    const int* const ids = sids + sl_cur * 8;
    const double ir = smat[sl_cur * 4 + 0], c2r = smat[sl_cur * 4 + 1];
    const double tau = smat[sl_cur * 4 + 2], irt = smat[sl_cur * 4 + 3];

    // ---- P1: Gauss values uq = B (x)3 U -> wA --------------------------------
    double* uq = scurv::vsweep3<N, TG, T_B>(A, us, wA, wB, tid);   // result in wA
    if constexpr (OPER) {
      // ---- P2: own face-node slices -> wB, then both trace sets to Gauss ----
      for (int t2 = tid; t2 < 6 * C * NF; t2 += TG) {
        const int f = t2 / (C * NF), rest = t2 - f * (C * NF);
        const int c = rest / NF, fn = rest - c * NF;
        wB[t2] = us[c * NODES + face_to_node<N>(f >> 1, f & 1, fn)];
      }
      __syncthreads();
      scurv::tsweep<N, 2, 0, 24, TG, T_B>(A, wB, wR, tid);
      __syncthreads();
      scurv::tsweep<N, 2, 1, 24, TG, T_B>(A, wR, wB, tid);
      __syncthreads();
      scurv::tsweep<N, 2, 0, 24, TG, T_B>(A, nbt, wR, tid);
      __syncthreads();
      scurv::tsweep<N, 2, 1, 24, TG, T_B>(A, wR, nbt, tid);
      __syncthreads();
      // ---- P3: strong half -> wR; face integrand over the neighbour traces --
      for (int pt = tid; pt < NODES; pt += TG) {
        double Gm[3][3];
#pragma unroll
        for (int m = 0; m < 3; ++m)
#pragma unroll
          for (int i = 0; i < 3; ++i) Gm[m][i] = ij[(m * 3 + i) * NODES + pt];
        const double jwp = jw[pt];
        double grad[3][C];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const int sm_ = m == 0 ? 1 : (m == 1 ? N : N * N);
          const int im = (pt / sm_) % N;
          const int base = pt - im * sm_;
          double row[N];
#pragma unroll
          for (int j = 0; j < N; ++j) row[j] = A.ctab[T_DCO + im * N + j];
#pragma unroll
          for (int c = 0; c < C; ++c) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) s = fma(row[j], uq[c * NODES + base + j * sm_], s);
            grad[m][c] = s;
          }
        }
        const double hv = 0.5 * jwp * ir, hp = 0.5 * jwp * c2r;
        double sv[3] = {0.0, 0.0, 0.0}, spp = 0.0;
#pragma unroll
        for (int m = 0; m < 3; ++m)
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            sv[i] = fma(Gm[m][i], grad[m][3], sv[i]);
            spp = fma(Gm[m][i], grad[m][i], spp);
          }
#pragma unroll
        for (int i = 0; i < 3; ++i) wR[i * NODES + pt] = hv * sv[i];
        wR[3 * NODES + pt] = hp * spp;
      }
      for (int t2 = tid; t2 < 6 * NF; t2 += TG) {
        const int f = t2 / NF, fn = t2 - f * NF;
        const int nbr = ids[f];
        double own[C], oth[C];
#pragma unroll
        for (int c = 0; c < C; ++c) own[c] = wB[(f * C + c) * NF + fn];
        if (nbr == -1) {
#pragma unroll
          for (int c = 0; c < 3; ++c) oth[c] = own[c];
          oth[3] = -own[3];
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) oth[c] = nbt[(f * C + c) * NF + fn];
        }
        const double* nrm_p = st + K::S_FN + f * 3 * NF + fn;
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
        const double fj = st[K::S_FJ + f * NF + fn];
#pragma unroll
        for (int i = 0; i < 3; ++i) nbt[(f * C + i) * NF + fn] = pv * nrm[i] * fj;
        nbt[(f * C + 3) * NF + fn] = pp * fj;
      }
      __syncthreads();
      // ---- P4: per direction m: weak flux tile -> wB, D_co^T along m and the
      //      face lifts (rows of B^{-1}) into wR; the last pass divides by JxW
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        for (int pt = tid; pt < NODES; pt += TG) {
          const double jwp = jw[pt];
          const double hv = 0.5 * jwp * ir, hp = 0.5 * jwp * c2r;
          const double pq = uq[3 * NODES + pt];
          double vg = 0.0;
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const double g = ij[(m * 3 + i) * NODES + pt];
            wB[i * NODES + pt] = -hv * g * pq;
            vg = fma(g, uq[i * NODES + pt], vg);
          }
          wB[3 * NODES + pt] = -hp * vg;
        }
        __syncthreads();
        const int sm_ = m == 0 ? 1 : (m == 1 ? N : N * N);
        for (int t2 = tid; t2 < VOL; t2 += TG) {
          const int c = t2 / NODES, pt = t2 - c * NODES;
          const int im = (pt / sm_) % N;
          const int base = pt - im * sm_;
          const double* src = wB + c * NODES + base;
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) s = fma(A.ctab[T_DCOT + im * N + j], src[j * sm_], s);
          double acc = wR[t2] + s;
          const int fn = node_to_face<N>(m, pt);
          const double l0 = A.ctab[T_BINV + 0 * N + im], l1 = A.ctab[T_BINV + (N - 1) * N + im];
          acc = fma(l0, nbt[((2 * m) * C + c) * NF + fn],
                    fma(l1, nbt[((2 * m + 1) * C + c) * NF + fn], acc));
          if (m == 2) acc /= jw[pt];
          wR[t2] = acc;
        }
        __syncthreads();
      }
      // ---- P5: W (GL) = B^{-1} (x)3 [R / JxW] -> wA (R keeps W at the Gauss points)
      double* wgl = scurv::vsweep3<N, TG, T_BINV>(A, wR, wA, wB, tid);
      if constexpr (!ADER) {
        // ---- operator outputs (coalesced) -----------------------------------
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          const int idx = tid + j * TG;
          if (idx < VOL) {
            const double v = wgl[idx];
            if (MODE == OUT_MINVK) {
              op.out[goff + idx] = v;
            } else if (MODE == OUT_RHS) {
              op.out[goff + idx] = -v;
            } else if (MODE == OUT_LSRK) {
              const double f = -v * op.dt;
              const double rr = read_r ? fma(op.a, rv[j], f) : f;
              op.r[goff + idx] = rr;
              op.u_out[goff + idx] = fma(op.b, rr, us[idx]);
            } else if (MODE == OUT_ADERB) {
              op.out[goff + idx] = rv[j] - v;
            }
          }
        }
      } else {
        // V = U - dt W
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
          const int idx = tid + j * TG;
          if (idx < VOL) A.t.v_out[goff + idx] = us[idx] - A.t.dt * wgl[idx];
        }
        __syncthreads();
      }
    }
    if constexpr (ADER) {
      // ---- Taylor loop at the Gauss points, compile-time plan ----------------
      double* cur = HDG ? wR : uq;
      double* nx = HDG ? wA : wR;
      double acc[N][RPL];
      constexpr TckPlan PL = sader::Plan<3, N, STRIDE, SHIFT>::P;
      scurv::run_plan<N, KC::REDLEN, STRIDE, SHIFT, RPL>(
          A, cur, nx, acc, st, ir, c2r, tid, std::make_integer_sequence<int, PL.n>{});
      // y = B^{-1} acc_k
      sader::acc_op<3, N, TG, 1, N - 1, TCK_LOAD, 0>(A.t, acc[N - 1], cur, tid);
      double* spare = (cur != wA && nx != wA) ? wA : ((cur != wB && nx != wB) ? wB : wR);
      scurv::tsweep<N, 3, 0, 4, TG, T_BINV>(A, cur, nx, tid);
      __syncthreads();
      scurv::tsweep<N, 3, 1, 4, TG, T_BINV>(A, nx, spare, tid);
      __syncthreads();
      scurv::tsweep<N, 3, 2, 4, TG, T_BINV>(A, spare, nx, tid);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        const int idx = tid + j * TG;
        if (idx < VOL) A.t.y[goff + idx] = nx[idx];
      }
    }
    // publish ids / material of tile nn, free the stage
    if (tid < 6) sids[sl_nn * 8 + tid] = idr;
    else if (tid >= 8 && tid < 12) smat[sl_nn * 4 + tid - 8] = matr;
    __syncthreads();
    buf ^= 1;
    ++it;
    tile = nxt;
    nxt = nn;
    nn = nnn;
  }
  sched_done(op.sched, tid == 0, pend, raw);
}

}  // namespace wk
