// Warp-group ADER kernel A for axis-aligned (Cartesian) affine cells:
// (ader_hdg) W = M^{-1} K U, V = U - dt W, y = TCK_shift(W);
// (ader)     y = TCK(U).                               (stepping.py:265-285)
//
// One group of TG threads owns one element (TG = 32 for n <= 5, 64 for
// n <= 8): no CTA-wide barriers, every step of the Taylor loop is a set of
// pencil sweeps inside the group's shared-memory tile:
//   * S (operator.py:286-306) on a Cartesian cell: v_m <- ir G_mm D p along m,
//     p <- c2r sum_m G_mm D v_m  -- pencils along each direction, the p share
//     accumulated in shared memory like the operator kernel (wk_group.cuh);
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
  static constexpr int TG = ((NF + 31) / 32) * 32;       // one element per group
  static constexpr int GPB = 1;                           // smem-heavy: 1 group / CTA
  static constexpr int TPB = TG * GPB;
  // per-group smem (doubles): U | nb/F | Rp | cur | nxt | mat | acc(...)
  static constexpr int G_U = 0;
  static constexpr int G_NB = C * NODES;
  static constexpr int G_RP = G_NB + 2 * D * 2 * NF;
  static constexpr int G_CUR = G_RP + NODES;
  static constexpr int G_NXT = G_CUR + C * NODES;
  static constexpr int G_MAT = G_NXT + C * NODES;
  static constexpr int G_ACC = G_MAT + kMatStride;
  __host__ __device__ static int group_doubles(int acc_len) { return (G_ACC + acc_len + 1) / 2 * 2; }
  __host__ __device__ static size_t bytes(int acc_len, int tab_len) {
    return sizeof(double) *
           (size_t)(GPB * group_doubles(acc_len) + N * N + 2 * N + GeoLayout<D>::STRIDE + tab_len);
  }
};

// S on a Cartesian cell at n points per direction, cur -> nxt.
template <int D, int N, int TG>
__device__ __forceinline__ void gader_apply_S(const double* cur, double* nxt, double* rp,
                                              const double* dm, int n, const double* geo,
                                              double ir, double c2r, int lane, int gid) {
  constexpr int C = D + 1, NODES = GroupCfg<D, N>::NODES;
  const int nf = D == 3 ? n * n : n;
  for (int m = 0; m < D; ++m) {
    const int sm = m == 0 ? 1 : (m == 1 ? n : n * n);
    const double gmm = geo[m * D + m];
    const double cv = ir * gmm, cp = c2r * gmm;
    for (int ln = lane; ln < nf; ln += TG) {
      // pencil along m through face position ln
      int b0;
      if (m == 0) b0 = ln * n;
      else if (m == 1) b0 = ln % n + (ln / n) * n * n;
      else b0 = ln;
      double pl[N], vl[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (j < n) {
          pl[j] = cur[D * NODES + b0 + j * sm];
          vl[j] = cur[m * NODES + b0 + j * sm];
        }
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if (i >= n) break;
        double ap = 0.0, av = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          if (j < n) {
            const double a = dm[i * n + j];
            ap = fma(a, pl[j], ap);
            av = fma(a, vl[j], av);
          }
        }
        const int node = b0 + i * sm;
        nxt[m * NODES + node] = cv * ap;
        const double s = cp * av;
        if (m == 0) rp[node] = s;
        else if (m < D - 1) rp[node] += s;
        else nxt[D * NODES + node] = rp[node] + s;
      }
    }
    group_sync<TG>(gid);
  }
}

// Resize every direction nf -> nt with an (nt x nf) matrix, cur -> nxt (the
// result ends in `cur` after the pointer swaps).
template <int D, int N, int TG>
__device__ __forceinline__ void gader_resize(double*& cur, double*& nxt, const double* mat,
                                             int nfr, int nto, int lane, int gid) {
  constexpr int C = D + 1, NODES = GroupCfg<D, N>::NODES;
  for (int m = 0; m < D; ++m) {
    int ein[3] = {1, 1, 1};
    for (int q = 0; q < D; ++q) ein[q] = q < m ? nto : nfr;
    // output extents: ein with direction m -> nto
    const int sm_in = m == 0 ? 1 : (m == 1 ? ein[0] : ein[0] * ein[1]);
    const int lines = (D == 3 ? ein[0] * ein[1] * ein[2] : ein[0] * ein[1]) / nfr;
    // input/output tensors share the line indexing of the other directions
    const int lo_ext = sm_in;            // product of extents below m
    for (int t = lane; t < C * lines; t += TG) {
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
    group_sync<TG>(gid);
    double* tt = cur; cur = nxt; nxt = tt;
  }
}

template <int D, int N, bool HDG>
__global__ void __launch_bounds__(GroupAderCfg<D, N>::TPB)
affine_group_ader_kernel(TckArgs T) {
  using K = GroupAderCfg<D, N>;
  using GLy = GeoLayout<D>;
  constexpr int C = K::C, NODES = K::NODES, NF = K::NF, TG = K::TG;
  const AffineArgs args = T.op;  // by value: no references into param space
  extern __shared__ __align__(16) double smem[];
  const int gdoubles = K::group_doubles(T.acc_len);
  double* const tabs = smem + K::GPB * gdoubles;
  double* const geo = tabs + N * N + 2 * N;
  double* const ttab = geo + GLy::STRIDE;
  const int tid = threadIdx.x;
  for (int i = tid; i < N * N + 2 * N; i += K::TPB) tabs[i] = args.tab[i];
  for (int i = tid; i < GLy::STRIDE; i += K::TPB) geo[i] = args.geo[i];
  for (int i = tid; i < T.tab_len; i += K::TPB) ttab[i] = T.tck_tab[i];
  __syncthreads();

  const int gid = tid / TG, lane = tid - gid * TG;
  double* const gs = smem + gid * gdoubles;
  double* const su = gs + K::G_U;
  double* const snb = gs + K::G_NB;
  double* const srp = gs + K::G_RP;
  double* cur = gs + K::G_CUR;
  double* nxt = gs + K::G_NXT;
  double* const smt = gs + K::G_MAT;
  double* const acc = gs + K::G_ACC;
  const long long e = args.e_begin + (long long)blockIdx.x * K::GPB + gid;
  if (e >= args.e_begin + args.E) return;

  // ---- stage U, material (and the neighbour faces for the HDG operator) ----
  {
    const double* gu = args.u + e * C * NODES;
    if (((e * C * NODES) & 1) == 0) {
      for (int i = 2 * lane; i < C * NODES; i += 2 * TG) {
        if (i + 1 < C * NODES) cp_async16(su + i, gu + i); else cp_async8(su + i, gu + i);
      }
    } else {
      for (int i = lane; i < C * NODES; i += TG) cp_async8(su + i, gu + i);
    }
    for (int i = lane; i < kMatStride; i += TG) cp_async8(smt + i, args.mat + e * kMatStride + i);
    if (HDG) {
#pragma unroll
      for (int f = 0; f < 2 * D; ++f) {
        const int m = f >> 1, sd = f & 1;
        const int nb = __ldg(args.nbr + e * 2 * D + f);
        for (int fn = lane; fn < NF; fn += TG) {
          double* dst = snb + f * 2 * NF + fn;
          if (nb >= 0) {
            const double* src = args.u + (long long)nb * C * NODES + face_to_node<N>(m, 1 - sd, fn);
            cp_async8(dst, src + m * NODES);
            cp_async8(dst + NF, src + D * NODES);
          } else if (nb <= -2) {
            const double* src = args.ghost + (long long)ghost_slot(nb) * C * NF + fn;
            cp_async8(dst, src + m * NF);
            cp_async8(dst + NF, src + D * NF);
          }
        }
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    group_sync<TG>(gid);
  }
  const double ir = smt[0], c2r = smt[1], tau = smt[2], irt = smt[3];

  if (HDG) {
    // ---- face integrands (v_m, p), in place --------------------------------
#pragma unroll
    for (int f = 0; f < 2 * D; ++f) {
      const int m = f >> 1, sd = f & 1;
      const int nb = __ldg(args.nbr + e * 2 * D + f);
      const double nm = geo[GLy::NORMAL + (m * 2 + sd) * D + m];
      const double fs = geo[GLy::FSCALE + m * 2 + sd];
      for (int fn = lane; fn < NF; fn += TG) {
        const double* uq = su + face_to_node<N>(m, sd, fn);
        const double vo = uq[m * NODES], po = uq[D * NODES];
        double* slot = snb + f * 2 * NF + fn;
        double vx, px;
        if (nb == -1) {
          vx = vo;
          px = -po;
        } else {
          vx = slot[0];
          px = slot[NF];
        }
        const double vn_o = nm * vo, vn_x = nm * vx;
        double pv = 0.5 * ir * px;
        double pp = 0.5 * c2r * vn_x;
        if (args.stab) {
          pv += 0.5 * irt * (vn_o - vn_x);
          pp += 0.5 * c2r * tau * (po - px);
        }
        slot[0] = pv * nm * fs;
        slot[NF] = pp * fs;
      }
    }
    group_sync<TG>(gid);
    // ---- W = M^{-1} K U by pencils; V = U - dt W to global, W -> cur ------
    const double* sA = tabs;
    const double* sL0 = tabs + N * N;
    const double* sL1 = sL0 + N;
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
      const double gmm = geo[m * D + m];
      const double cv = ir * gmm, cp = c2r * gmm;
      for (int fn = lane; fn < NF; fn += TG) {
        const int nb0 = pencil_base<N>(m, fn);
        double pl[N], vl[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          pl[i] = su[D * NODES + nb0 + i * sm];
          vl[i] = su[m * NODES + nb0 + i * sm];
        }
        const double* f0 = snb + (2 * m) * 2 * NF + fn;
        const double fv0 = f0[0], fp0 = f0[NF], fv1 = f0[2 * NF], fp1 = f0[3 * NF];
        const long long gb = e * C * NODES + nb0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double ap = 0.0, av = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            const double a = sA[i * N + j];
            ap = fma(a, pl[j], ap);
            av = fma(a, vl[j], av);
          }
          const double l0 = sL0[i], l1 = sL1[i];
          const double wv = fma(cv, ap, fma(l0, fv0, l1 * fv1));
          double wp = fma(cp, av, fma(l0, fp0, l1 * fp1));
          const int node = nb0 + i * sm;
          cur[m * NODES + node] = wv;
          T.v_out[gb + m * NODES + i * sm] = vl[i] - T.dt * wv;
          if (m == 0) {
            srp[node] = wp;
          } else if (m < D - 1) {
            srp[node] += wp;
          } else {
            wp += srp[node];
            cur[D * NODES + node] = wp;
            T.v_out[gb + D * NODES + i * sm] = pl[i] - T.dt * wp;
          }
        }
      }
      group_sync<TG>(gid);
    }
  } else {
    for (int i = lane; i < C * NODES; i += TG) cur[i] = su[i];
    group_sync<TG>(gid);
  }

  // ---- Taylor loop program ------------------------------------------------
  for (int op = 0; op < T.nops; ++op) {
    const int code = __ldg(T.prog + 4 * op + 0);
    const int a0 = __ldg(T.prog + 4 * op + 1);
    const int a1 = __ldg(T.prog + 4 * op + 2);
    const int a2 = __ldg(T.prog + 4 * op + 3);
    if (code == TCK_S) {
      gader_apply_S<D, N, TG>(cur, nxt, srp, ttab + a1, a0, geo, ir, c2r, lane, gid);
      double* t = cur; cur = nxt; nxt = t;
    } else if (code == TCK_RESIZE) {
      gader_resize<D, N, TG>(cur, nxt, ttab + a2, a0, a1, lane, gid);
    } else {
      const double w = __ldg(T.weights + op);
      const int nn = npow<D>(a1);
      for (int t = lane; t < C * nn; t += TG) {
        const int c = t / nn, pt = t - c * nn;
        double* slot = acc + a0 + c * nn + pt;
        double* cv = cur + c * NODES + pt;
        if (code == TCK_ACC_SET) *slot = w * *cv;
        else if (code == TCK_ACC_ADD) *slot = *slot + w * *cv;
        else *cv = *slot;
      }
      group_sync<TG>(gid);
    }
  }
  // slot 0 holds acc_k (GL) = M^{-1} T
  double* gy = T.y + e * C * NODES;
  for (int i = lane; i < C * NODES; i += TG) gy[i] = acc[i];
}

}  // namespace wk
