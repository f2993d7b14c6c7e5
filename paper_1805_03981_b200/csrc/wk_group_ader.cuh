// ADER kernel A for axis-aligned (Cartesian) affine cells:
// (ader_hdg) W = M^{-1} K U, V = U - dt W, y = TCK_shift(W);
// (ader)     y = TCK(U).                               (stepping.py:265-285)
//
// One CTA owns one element.  Every step of the Taylor loop is a set of pencil
// sweeps over the element's shared-memory tile, with TWO lanes per pencil
// (one produces the v_m result, the other the pressure share), so that even
// the 8^3 tiles of config 4 keep 4 warps of independent FMA chains:
//   * S (operator.py:286-306) on a Cartesian cell: v_m <- ir G_mm D p along m,
//     p <- c2r sum_m G_mm D v_m;  the p shares accumulate in shared memory;
//   * resize (projection / interpolation, operator.py:308-325): one pass per
//     direction, a lane per (component, line);
//   * accumulators: element-wise.
// The op program is the one wk_tck.cuh interprets (built by get_program in
// wk_abi.cu, full degree in the GL basis); y = acc_k is written in GL.
#pragma once
#include "wk_group.cuh"
#include "wk_tck.cuh"

namespace wk {

template <int D, int N>
struct GroupAderCfg {
  using G = GroupCfg<D, N>;
  static constexpr int C = D + 1, NODES = G::NODES, NF = G::NF;
  static constexpr int TE0 = ((2 * NF + 31) / 32) * 32;
  static constexpr int TE = TE0 > 256 ? 256 : TE0;        // threads per element (= CTA)
  static constexpr int GPB = 1;
  static constexpr int TPB = TE;
  // smem (doubles): A (U, later scratch) | B | nb/F | Rp | mat | acc | tables
  static constexpr int G_A = 0;
  static constexpr int G_B = C * NODES;
  static constexpr int G_NB = 2 * C * NODES;
  static constexpr int G_RP = G_NB + 2 * D * 2 * NF;
  static constexpr int G_MAT = G_RP + NODES;
  static constexpr int G_ACC = G_MAT + kMatStride;
  __host__ __device__ static int off_tab(int acc_len) { return (G_ACC + acc_len + 1) / 2 * 2; }
  __host__ __device__ static size_t bytes(int acc_len, int tab_len) {
    return sizeof(double) *
           (size_t)(off_tab(acc_len) + N * N + 2 * N + GeoLayout<D>::STRIDE + tab_len);
  }
};

// S on a Cartesian cell at NN points per direction (compile time), cur -> nxt
// (two lanes per pencil: half 0 -> v_m, half 1 -> p share).
template <int D, int N, int TE, int NN>
__device__ __forceinline__ void gader_apply_S_ct(const double* cur, double* nxt, double* rp,
                                                 const double* dm, const double* geo,
                                                 double ir, double c2r, int tid) {
  constexpr int NODES = GroupCfg<D, N>::NODES;
  constexpr int NFF = D == 3 ? NN * NN : NN;
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? NN : NN * NN);
    const double gmm = geo[m * D + m];
    for (int t = tid; t < 2 * NFF; t += TE) {
      const int half = t >= NFF ? 1 : 0;
      const int ln = t - half * NFF;
      const int b0 = m == 0 ? ln * NN : (m == 1 ? ln % NN + (ln / NN) * NN * NN : ln);
      // half 0 differentiates p (-> v_m), half 1 differentiates v_m (-> p)
      const double* src = cur + (half ? m : D) * NODES + b0;
      double x[NN];
#pragma unroll
      for (int j = 0; j < NN; ++j) x[j] = src[j * sm];
      const double coef = (half ? c2r : ir) * gmm;
#pragma unroll
      for (int i = 0; i < NN; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NN; ++j) acc = fma(dm[i * NN + j], x[j], acc);
        const int node = b0 + i * sm;
        acc *= coef;
        if (!half) {
          nxt[m * NODES + node] = acc;
        } else if (m == 0) {
          rp[node] = acc;
        } else if (m < D - 1) {
          rp[node] += acc;
        } else {
          nxt[D * NODES + node] = rp[node] + acc;
        }
      }
    }
    __syncthreads();
  }
}

// ---- FP64 tensor-core (DMMA, mma.sync m8n8k4) versions ----------------
// ncu on config 4 showed the CUDA-core sweeps issue-bound (one shared-memory
// load of a matrix entry per DFMA).  A warp-wide m8n8k4 DMMA does 256 FMAs
// per instruction with the 1-D matrix held as two A fragments in registers:
// Y[i][p] = sum_j M[i][j] X[j][p] for 8 pencils p at a time (zero-padded to
// 8 rows / 4k columns).  Fragment layout (verified by tools/dmma_check.cu):
// A lane l = M[l>>2][l&3], B lane l = X[l&3][l>>2], C lane l = Y[l>>2][2(l&3)+{0,1}].
// (dmma884: wk_common.cuh)

template <int N, int NN>
__device__ __forceinline__ int pbase(int m, int p) {
  return m == 0 ? p * NN : (m == 1 ? p % NN + (p / NN) * NN * NN : p);
}

// n = 8, d = 3: chunks of 8 pencils are affine in memory for every direction,
// so the fragment addresses need no division at all.
template <int D, int N, int TE>
__device__ __forceinline__ void gader_apply_S_mma8(const double* cur, double* nxt, double* rp,
                                                   const double* dm, const double* geo,
                                                   double ir, double c2r, int tid) {
  constexpr int NODES = GroupCfg<D, N>::NODES;
  constexpr int NW = TE / 32;
  const int lane = tid & 31, warp = tid >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const double a0 = dm[ar * 8 + ac], a1 = dm[ar * 8 + 4 + ac];
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? 8 : 64);
    const int ps = m == 0 ? 8 : 1;            // stride between the chunk's pencils
    const double gmm = geo[m * D + m];
    for (int u = warp; u < 16; u += NW) {     // 8 chunks x 2 halves
      const int half = u >> 3, c = u & 7;
      const int cb = m == 2 ? 8 * c : 64 * c;
      const double* src = cur + (half ? m : D) * NODES + cb;
      const int bo = ar * ps + ac * sm;
      double c0 = 0.0, c1 = 0.0;
      dmma884(c0, c1, a0, src[bo]);
      dmma884(c0, c1, a1, src[bo + 4 * sm]);
      const double coef = (half ? c2r : ir) * gmm;
      const int n0 = cb + (2 * ac) * ps + ar * sm;
      const int n1 = n0 + ps;
      const double v0 = c0 * coef, v1 = c1 * coef;
      if (!half) {
        nxt[m * NODES + n0] = v0;
        nxt[m * NODES + n1] = v1;
      } else if (m == 0) {
        rp[n0] = v0;
        rp[n1] = v1;
      } else if (m == 1) {
        rp[n0] += v0;
        rp[n1] += v1;
      } else {
        nxt[D * NODES + n0] = rp[n0] + v0;
        nxt[D * NODES + n1] = rp[n1] + v1;
      }
    }
    __syncthreads();
  }
}

template <int D, int N, int TE, int NN>
__device__ __forceinline__ void gader_apply_S_mma(const double* cur, double* nxt, double* rp,
                                                  const double* dm, const double* geo,
                                                  double ir, double c2r, int tid) {
  constexpr int NODES = GroupCfg<D, N>::NODES;
  constexpr int NFF = D == 3 ? NN * NN : NN;
  constexpr int CH = (NFF + 7) / 8, KS = (NN + 3) / 4, NW = TE / 32;
  const int lane = tid & 31, warp = tid >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  double af[KS];
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int j = 4 * kk + ac;
    af[kk] = (ar < NN && j < NN) ? dm[ar * NN + j] : 0.0;
  }
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? NN : NN * NN);
    const double gmm = geo[m * D + m];
    for (int u = warp; u < 2 * CH; u += NW) {
      const int half = u >= CH ? 1 : 0;
      const int p0 = (u - half * CH) * 8;
      const double* src = cur + (half ? m : D) * NODES;
      const int pb = p0 + ar;
      const bool pv = pb < NFF;
      const int bb = pv ? pbase<N, NN>(m, pb) : 0;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int j = 4 * kk + ac;
        const double b = (pv && j < NN) ? src[bb + j * sm] : 0.0;
        dmma884(c0, c1, af[kk], b);
      }
      if (ar < NN) {
        const double coef = (half ? c2r : ir) * gmm;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int p = p0 + 2 * ac + t;
          if (p >= NFF) continue;
          const int node = pbase<N, NN>(m, p) + ar * sm;
          const double val = (t ? c1 : c0) * coef;
          if (!half) {
            nxt[m * NODES + node] = val;
          } else if (m == 0) {
            rp[node] = val;
          } else if (m < D - 1) {
            rp[node] += val;
          } else {
            nxt[D * NODES + node] = rp[node] + val;
          }
        }
      }
    }
    __syncthreads();
  }
}

template <int D, int N, int TE, int NF_, int NT_>
__device__ __forceinline__ void gader_resize_mma(double*& cur, double*& nxt, const double* mat,
                                                 int tid) {
  constexpr int C = D + 1, NODES = GroupCfg<D, N>::NODES;
  constexpr int KS = (NF_ + 3) / 4, NW = TE / 32;
  const int lane = tid & 31, warp = tid >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  double af[KS];
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int j = 4 * kk + ac;
    af[kk] = (ar < NT_ && j < NF_) ? mat[ar * NF_ + j] : 0.0;
  }
#pragma unroll
  for (int m = 0; m < D; ++m) {
    const int lo_ext = m == 0 ? 1 : (m == 1 ? NT_ : NT_ * NT_);
    const int hi_ext = D == 3 ? (m == 0 ? NF_ * NF_ : (m == 1 ? NF_ : 1)) : (m == 0 ? NF_ : 1);
    const int lines = lo_ext * hi_ext;
    const int ch = (lines + 7) / 8;
    for (int u = warp; u < C * ch; u += NW) {
      const int c = u / ch;
      const int p0 = (u - c * ch) * 8;
      const int pb = p0 + ar;
      const bool pv = pb < lines;
      const int hb = pv ? pb / lo_ext : 0, lb = pv ? pb - hb * lo_ext : 0;
      const double* src = cur + c * NODES + lb + hb * lo_ext * NF_;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int j = 4 * kk + ac;
        const double b = (pv && j < NF_) ? src[j * lo_ext] : 0.0;
        dmma884(c0, c1, af[kk], b);
      }
      if (ar < NT_) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int p = p0 + 2 * ac + t;
          if (p >= lines) continue;
          const int h = p / lo_ext, l = p - h * lo_ext;
          nxt[c * NODES + l + h * lo_ext * NT_ + ar * lo_ext] = t ? c1 : c0;
        }
      }
    }
    __syncthreads();
    double* tt = cur; cur = nxt; nxt = tt;
  }
}

template <int D, int N, int TE>
__device__ __forceinline__ void gader_apply_S(const double* cur, double* nxt, double* rp,
                                              const double* dm, int n, const double* geo,
                                              double ir, double c2r, int tid) {
  switch (n) {
#define WK_S_CASE(k) \
  case k:            \
    if constexpr (k == 8 && N == 8 && D == 3) gader_apply_S_mma8<D, N, TE>(cur, nxt, rp, dm, geo, ir, c2r, tid); \
    else if constexpr (k <= N && k <= 8 && N >= 7) gader_apply_S_mma<D, N, TE, k>(cur, nxt, rp, dm, geo, ir, c2r, tid); \
    else if constexpr (k <= N) gader_apply_S_ct<D, N, TE, k>(cur, nxt, rp, dm, geo, ir, c2r, tid); \
    return;
    WK_S_CASE(1) WK_S_CASE(2) WK_S_CASE(3) WK_S_CASE(4) WK_S_CASE(5) WK_S_CASE(6)
    WK_S_CASE(7) WK_S_CASE(8) WK_S_CASE(9)
#undef WK_S_CASE
  }
}

// Resize every direction NF_ -> NT_ (compile time) with an (NT_ x NF_) matrix;
// result in cur.
template <int D, int N, int TE, int NF_, int NT_>
__device__ __forceinline__ void gader_resize_ct(double*& cur, double*& nxt, const double* mat,
                                                int tid) {
  constexpr int C = D + 1, NODES = GroupCfg<D, N>::NODES;
#pragma unroll
  for (int m = 0; m < D; ++m) {
    // extents before this pass: directions < m already resized
    const int lo_ext = m == 0 ? 1 : (m == 1 ? NT_ : NT_ * NT_);
    const int hi_ext = D == 3 ? (m == 0 ? NF_ * NF_ : (m == 1 ? NF_ : 1)) : (m == 0 ? NF_ : 1);
    const int lines = lo_ext * hi_ext;
    for (int c = 0; c < C; ++c) {
      for (int l = tid; l < lines; l += TE) {
        const int hi = l / lo_ext, lo = l - hi * lo_ext;
        const double* src = cur + c * NODES + lo + hi * lo_ext * NF_;
        double x[NF_];
#pragma unroll
        for (int j = 0; j < NF_; ++j) x[j] = src[j * lo_ext];
        double* dst = nxt + c * NODES + lo + hi * lo_ext * NT_;
#pragma unroll
        for (int i = 0; i < NT_; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < NF_; ++j) acc = fma(mat[i * NF_ + j], x[j], acc);
          dst[i * lo_ext] = acc;
        }
      }
    }
    __syncthreads();
    double* tt = cur; cur = nxt; nxt = tt;
  }
}

// generic runtime-extent fallback
template <int D, int N, int TE>
__device__ __forceinline__ void gader_resize_rt(double*& cur, double*& nxt, const double* mat,
                                                int nfr, int nto, int tid) {
  constexpr int C = D + 1, NODES = GroupCfg<D, N>::NODES;
  for (int m = 0; m < D; ++m) {
    int ein[3] = {1, 1, 1};
    for (int q = 0; q < D; ++q) ein[q] = q < m ? nto : nfr;
    const int lo_ext = m == 0 ? 1 : (m == 1 ? ein[0] : ein[0] * ein[1]);
    const int lines = (D == 3 ? ein[0] * ein[1] * ein[2] : ein[0] * ein[1]) / nfr;
    const UDiv dl((unsigned)lines), dlo((unsigned)lo_ext);
    for (int t = tid; t < C * lines; t += TE) {
      const int c = (int)dl.div((unsigned)t), l = t - c * lines;
      const int hi = (int)dlo.div((unsigned)l), lo = l - hi * lo_ext;
      const double* src = cur + c * NODES + lo + hi * lo_ext * nfr;
      double x[N];
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (j < nfr) x[j] = src[j * lo_ext];
      double* dst = nxt + c * NODES + lo + hi * lo_ext * nto;
      for (int i = 0; i < nto; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j)
          if (j < nfr) acc = fma(mat[i * nfr + j], x[j], acc);
        dst[i * lo_ext] = acc;
      }
    }
    __syncthreads();
    double* tt = cur; cur = nxt; nxt = tt;
  }
}

template <int D, int N, int TE>
__device__ __forceinline__ void gader_resize(double*& cur, double*& nxt, const double* mat,
                                             int nfr, int nto, int tid) {
  // the reduction schedules only step by 1..3 degrees (kernels.py:279-302)
  switch (nfr * 16 + nto) {
#define WK_R(a, b)                                                                  \
  case a * 16 + b:                                                                  \
    if constexpr (a <= N && b <= N && a <= 8 && b <= 8 && N >= 7) return gader_resize_mma<D, N, TE, a, b>(cur, nxt, mat, tid); \
    else if constexpr (a <= N && b <= N) return gader_resize_ct<D, N, TE, a, b>(cur, nxt, mat, tid); \
    break;
#define WK_R3(n) WK_R(n, n - 1) WK_R(n - 1, n)
    WK_R3(2) WK_R3(3) WK_R3(4) WK_R3(5) WK_R3(6) WK_R3(7) WK_R3(8) WK_R3(9)
    WK_R(3, 1) WK_R(1, 3) WK_R(4, 2) WK_R(2, 4) WK_R(5, 3) WK_R(3, 5) WK_R(6, 4) WK_R(4, 6)
    WK_R(7, 5) WK_R(5, 7) WK_R(8, 6) WK_R(6, 8) WK_R(9, 7) WK_R(7, 9)
    WK_R(4, 1) WK_R(1, 4) WK_R(5, 2) WK_R(2, 5) WK_R(6, 3) WK_R(3, 6) WK_R(7, 4) WK_R(4, 7)
    WK_R(8, 5) WK_R(5, 8) WK_R(9, 6) WK_R(6, 9)
#undef WK_R3
#undef WK_R
  }
  gader_resize_rt<D, N, TE>(cur, nxt, mat, nfr, nto, tid);
}

template <int D, int N, bool HDG>
__global__ void __launch_bounds__(GroupAderCfg<D, N>::TE)
affine_group_ader_kernel(const __grid_constant__ TckArgs T) {
  using K = GroupAderCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, TE = K::TE;
  const AffineArgs args = T.op;  // by value: no references into param space
  extern __shared__ __align__(16) double smem[];
  double* const sa = smem + K::G_A;
  double* const sb = smem + K::G_B;
  double* const snb = smem + K::G_NB;
  double* const srp = smem + K::G_RP;
  double* const smt = smem + K::G_MAT;
  double* const acc = smem + K::G_ACC;
  double* const tabs = smem + K::off_tab(T.acc_len);
  double* const geo = tabs + N * N + 2 * N;
  double* const ttab = geo + GLy::STRIDE;
  const int tid = threadIdx.x;
  const long long e = args.e_begin + blockIdx.x;
  if (e >= args.e_begin + args.E) return;
  for (int i = tid; i < N * N + 2 * N; i += TE) tabs[i] = args.tab[i];
  for (int i = tid; i < GLy::STRIDE; i += TE) geo[i] = args.geo[i];
  for (int i = tid; i < T.tab_len; i += TE) ttab[i] = T.tck_tab[i];

  // ---- stage U, material, neighbour (v_m, p) face values -------------------
  {
    const double* gu = args.u + e * C * NODES;
    if (((e * C * NODES) & 1) == 0) {
      for (int i = 2 * tid; i < C * NODES; i += 2 * TE) {
        if (i + 1 < C * NODES) cp_async16(sa + i, gu + i); else cp_async8(sa + i, gu + i);
      }
    } else {
      for (int i = tid; i < C * NODES; i += TE) cp_async8(sa + i, gu + i);
    }
    for (int i = tid; i < kMatStride; i += TE) cp_async8(smt + i, args.mat + e * kMatStride + i);
    if (HDG) {
      for (int t = tid; t < 2 * D * NF; t += TE) {
        const int f = t / NF, fn = t - (t / NF) * NF;
        const int m = f >> 1, sd = f & 1;
        const int nb = __ldg(args.nbr + e * 2 * D + f);
        WK_CHECK_NBR(args, nb);
        double* dst = snb + f * 2 * NF + fn;
        if (nb >= 0) {
          const double* src = args.u + (long long)nb * C * NODES + face_to_node<N>(m, 1 - sd, fn);
          cp_async8(dst, src + m * NODES);
          cp_async8(dst + NF, src + D * NODES);
        } else if (args.has_ghost && nb <= -2) {
          const double* src = args.ghost + (long long)ghost_slot(nb) * C * NF + fn;
          cp_async8(dst, src + m * NF);
          cp_async8(dst + NF, src + D * NF);
        }
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
  }
  const double ir = smt[0], c2r = smt[1], tau = smt[2], irt = smt[3];
  double* cur;
  double* nxt;

  if (HDG) {
    // ---- face integrands (v_m, p), in place --------------------------------
    for (int t = tid; t < 2 * D * NF; t += TE) {
      const int f = t / NF, fn = t - (t / NF) * NF;
      const int m = f >> 1, sd = f & 1;
      const int nb = __ldg(args.nbr + e * 2 * D + f);
      const double* uq = sa + face_to_node<N>(m, sd, fn);
      const double vo = uq[m * NODES], po = uq[D * NODES];
      double* slot = snb + f * 2 * NF + fn;
      const bool wall = nb == -1;
      double fv, fp;
      cart_face_flux(vo, po, wall ? vo : slot[0], wall ? -po : slot[NF],
                     geo[GLy::NORMAL + (m * 2 + sd) * D + m], geo[GLy::FSCALE + m * 2 + sd],
                     ir, c2r, tau, irt, args.stab, fv, fp);
      slot[0] = fv;
      slot[NF] = fp;
    }
    __syncthreads();
    // ---- W = M^{-1} K U (two lanes per pencil) into B; V = U - dt W -------
    const double* sA = tabs;
    const double* sL0 = tabs + N * N;
    const double* sL1 = sL0 + N;
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
      const double gmm = geo[m * D + m];
      for (int t = tid; t < 2 * NF; t += TE) {
        const int half = t >= NF ? 1 : 0;
        const int fn = t - half * NF;
        const int nb0 = pencil_base<N>(m, fn);
        const double* src = sa + (half ? m : D) * NODES + nb0;
        double x[N];
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] = src[j * sm];
        const double* f0 = snb + (2 * m) * 2 * NF + fn + (half ? NF : 0);
        const double g0 = f0[0], g1 = f0[2 * NF];   // face value (v or p comp) at both ends
        const double coef = (half ? c2r : ir) * gmm;
        const long long gb = e * C * NODES + nb0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) s = fma(sA[i * N + j], x[j], s);
          const double w = fma(coef, s, fma(sL0[i], g0, sL1[i] * g1));
          const int node = nb0 + i * sm;
          if (!half) {
            sb[m * NODES + node] = w;
            T.v_out[gb + m * NODES + i * sm] = sa[m * NODES + node] - T.dt * w;
          } else if (m == 0) {
            srp[node] = w;
          } else if (m < D - 1) {
            srp[node] += w;
          } else {
            const double wp = srp[node] + w;
            sb[D * NODES + node] = wp;
            T.v_out[gb + D * NODES + i * sm] = sa[D * NODES + node] - T.dt * wp;
          }
        }
      }
      __syncthreads();
    }
    cur = sb;
    nxt = sa;
  } else {
    cur = sa;
    nxt = sb;
  }

  // ---- Taylor loop program ------------------------------------------------
  for (int op = 0; op < T.nops; ++op) {
    const int code = __ldg(T.prog + 4 * op + 0);
    const int a0 = __ldg(T.prog + 4 * op + 1);
    const int a1 = __ldg(T.prog + 4 * op + 2);
    const int a2 = __ldg(T.prog + 4 * op + 3);
    if (code == TCK_S) {
      gader_apply_S<D, N, TE>(cur, nxt, srp, ttab + a1, a0, geo, ir, c2r, tid);
      double* t = cur; cur = nxt; nxt = t;
    } else if (code == TCK_RESIZE) {
      gader_resize<D, N, TE>(cur, nxt, ttab + a2, a0, a1, tid);
    } else {
      const double w = T.w[op];
      const int nn = npow<D>(a1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double* slot = acc + a0 + c * nn;
        double* cv = cur + c * NODES;
        if (code == TCK_ACC_SET) {
          for (int pt = tid; pt < nn; pt += TE) slot[pt] = w * cv[pt];
        } else if (code == TCK_ACC_ADD) {
          for (int pt = tid; pt < nn; pt += TE) slot[pt] = slot[pt] + w * cv[pt];
        } else {
          for (int pt = tid; pt < nn; pt += TE) cv[pt] = slot[pt];
        }
      }
      __syncthreads();
    }
  }
  // slot 0 holds acc_k (GL) = M^{-1} T
  double* gy = T.y + e * C * NODES;
  for (int i = tid; i < C * NODES; i += TE) gy[i] = acc[i];
}

}  // namespace wk
