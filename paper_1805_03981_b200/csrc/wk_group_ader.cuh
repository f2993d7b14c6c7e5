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

// S on a Cartesian cell at n points per direction, cur -> nxt (two lanes per
// pencil: half 0 -> v_m, half 1 -> p share).
template <int D, int N, int TE>
__device__ __forceinline__ void gader_apply_S(const double* cur, double* nxt, double* rp,
                                              const double* dm, int n, const double* geo,
                                              double ir, double c2r, int tid) {
  constexpr int NODES = GroupCfg<D, N>::NODES;
  const int nf = D == 3 ? n * n : n;
  for (int m = 0; m < D; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? n : n * n);
    const double gmm = geo[m * D + m];
    for (int t = tid; t < 2 * nf; t += TE) {
      const int half = t >= nf ? 1 : 0;
      const int ln = t - half * nf;
      int b0;
      if (m == 0) b0 = ln * n;
      else if (m == 1) b0 = ln % n + (ln / n) * n * n;
      else b0 = ln;
      // half 0 differentiates p (-> v_m), half 1 differentiates v_m (-> p)
      const double* src = cur + (half ? m : D) * NODES + b0;
      double x[N];
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (j < n) x[j] = src[j * sm];
      const double coef = (half ? c2r : ir) * gmm;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if (i >= n) break;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j)
          if (j < n) s = fma(dm[i * n + j], x[j], s);
        const int node = b0 + i * sm;
        s *= coef;
        if (!half) {
          nxt[m * NODES + node] = s;
        } else if (m == 0) {
          rp[node] = s;
        } else if (m < D - 1) {
          rp[node] += s;
        } else {
          nxt[D * NODES + node] = rp[node] + s;
        }
      }
    }
    __syncthreads();
  }
}

// Resize every direction nfr -> nto with an (nto x nfr) matrix; result in cur.
template <int D, int N, int TE>
__device__ __forceinline__ void gader_resize(double*& cur, double*& nxt, const double* mat,
                                             int nfr, int nto, int tid) {
  constexpr int C = D + 1, NODES = GroupCfg<D, N>::NODES;
  for (int m = 0; m < D; ++m) {
    int ein[3] = {1, 1, 1};
    for (int q = 0; q < D; ++q) ein[q] = q < m ? nto : nfr;
    const int lo_ext = m == 0 ? 1 : (m == 1 ? ein[0] : ein[0] * ein[1]);
    const int lines = (D == 3 ? ein[0] * ein[1] * ein[2] : ein[0] * ein[1]) / nfr;
    for (int t = tid; t < C * lines; t += TE) {
      const int c = t / lines, l = t - c * lines;
      const int lo = l % lo_ext, hi = l / lo_ext;
      const double* src = cur + c * NODES + lo + hi * lo_ext * nfr;
      double x[N];
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (j < nfr) x[j] = src[j * lo_ext];
      double* dst = nxt + c * NODES + lo + hi * lo_ext * nto;
      for (int i = 0; i < nto; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j)
          if (j < nfr) s = fma(mat[i * nfr + j], x[j], s);
        dst[i * lo_ext] = s;
      }
    }
    __syncthreads();
    double* tt = cur; cur = nxt; nxt = tt;
  }
}

template <int D, int N, bool HDG>
__global__ void __launch_bounds__(GroupAderCfg<D, N>::TE)
affine_group_ader_kernel(TckArgs T) {
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
      const double w = __ldg(T.weights + op);
      const int nn = npow<D>(a1);
      for (int t = tid; t < C * nn; t += TE) {
        const int c = t / nn, pt = t - c * nn;
        double* slot = acc + a0 + c * nn + pt;
        double* cv = cur + c * NODES + pt;
        if (code == TCK_ACC_SET) *slot = w * *cv;
        else if (code == TCK_ACC_ADD) *slot = *slot + w * *cv;
        else *cv = *slot;
      }
      __syncthreads();
    }
  }
  // slot 0 holds acc_k (GL) = M^{-1} T
  double* gy = T.y + e * C * NODES;
  for (int i = tid; i < C * NODES; i += TE) gy[i] = acc[i];
}

}  // namespace wk
