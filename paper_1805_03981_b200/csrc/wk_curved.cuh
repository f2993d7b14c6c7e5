// Curved-geometry (per-point metric) kernels: the reference's quadrature
// formulation evaluated element-by-element in shared memory.
//
// Reference: apply_K split form + face terms (operator.py:149-246) with the
// per-point GeometryCache arrays (mesh.py:162-188), fused with the inverse
// mass (operator.py:250-258):
//
//   K u        = B^T(x)d  R                       (R: quadrature-space residual)
//   M^{-1} K u = B^{-1}(x)d [ R / JxW ]           since B^{-T} B^T = I
//
// R collects the strong half  1/2 JxW S u  at the Gauss points, the weak half
// -1/2 sum_m D_co,m^T (JxW flux_m(u)) and the face integrand lifted into the
// Gauss basis with the GL-endpoint row of B^{-1} (B^T of that row is the unit
// face-node vector the reference adds into, operator.py:241-246).
//
// One element per CTA; 4d sweeps x (d+1) components of n^{d+1} FMAs plus
// per-point metric math.  Used for BASELINE config 3 (degree-5 curved map) and
// any non-affine (e.g. deformed multilinear) mesh.
#pragma once
#include "wk_affine.cuh"
#include "wk_tck.cuh"
#include "wk_group_ader.cuh"

namespace wk {

enum { OUT_K = 4 };  // extra curved output mode: out = K u

struct CurvedArgs {
  const double* inv_jac;              // (E, d, d, n^d)   degree-k Gauss points
  const double* jxw;                  // (E, n^d)
  const double* fnormal[6];           // (E, d, n^{d-1})  per face 2m+s
  const double* fjxw[6];              // (E, n^{d-1})
  const double* ctab;                 // B, Binv, Dco, DcoT, BT  (5 n^2)
  const double* invjac_deg[kMaxN];    // per degree q <= k (TCK), may be null
  int y_mode;                         // TCK output: 0 -> B^{-1} acc, 1 -> B^T (JxW acc)
};

template <int D, int N>
struct CShape {
  static constexpr int C = D + 1;
  static constexpr int NODES = D == 3 ? N * N * N : N * N;
  static constexpr int NF = D == 3 ? N * N : N;
  static constexpr int TPB = ((NODES + 31) / 32) * 32 < 64 ? 64 : ((NODES + 31) / 32) * 32;
  // smem (doubles)
  static constexpr int VOL = C * NODES;
  static constexpr int FACE = 2 * D * C * NF;
  static constexpr int TAB = 5 * N * N;
  // us, uq, tq, R, fl(D x VOL), nb, ftr, ntr, ftmp, tab
  static constexpr int OFF_US = 0;
  static constexpr int OFF_UQ = OFF_US + VOL;
  static constexpr int OFF_TQ = OFF_UQ + VOL;
  static constexpr int OFF_R = OFF_TQ + VOL;
  static constexpr int OFF_FL = OFF_R + VOL;
  static constexpr int OFF_NB = OFF_FL + D * VOL;
  static constexpr int OFF_FTR = OFF_NB + FACE;
  static constexpr int OFF_NTR = OFF_FTR + FACE;
  static constexpr int OFF_FTMP = OFF_NTR + FACE;
  static constexpr int OFF_TAB = OFF_FTMP + FACE;
  static constexpr int TOTAL = OFF_TAB + TAB;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
};

// Block-cooperative square sweep along direction M (compile time) over
// `ncomp` blocks of a tensor with N points per direction (stride `cstride`
// between blocks).  One thread per (block, line): the line's N inputs in
// registers, N outputs, index arithmetic once per line.
template <int D, int N, int M>
__device__ __forceinline__ void csweep(const double* in, double* out, const double* mat,
                                       int ncomp, int cstride, int npts) {
  constexpr int sm = M == 0 ? 1 : (M == 1 ? N : N * N);
  const int lines = npts / N;
  for (int t = threadIdx.x; t < ncomp * lines; t += blockDim.x) {
    const int c = t / lines, l = t - c * lines;
    // line l enumerates the other directions; base node with i_M = 0
    const int lo = l % sm, hi = l / sm;
    const int base = lo + hi * sm * N;
    const double* src = in + c * cstride + base;
    double x[N];
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = src[j * sm];
    double* dst = out + c * cstride + base;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) s = fma(mat[i * N + j], x[j], s);
      dst[i * sm] = s;
    }
  }
}

// Apply `mat` along every direction of a volume tensor: src preserved, result
// pointer returned (ping-pong between a and b).
template <int D, int N>
__device__ __forceinline__ double* csweep_all(const double* src, double* a, double* b,
                                              const double* mat, int ncomp) {
  constexpr int NODES = CShape<D, N>::NODES;
  csweep<D, N, 0>(src, a, mat, ncomp, NODES, NODES);
  __syncthreads();
  csweep<D, N, 1>(a, b, mat, ncomp, NODES, NODES);
  __syncthreads();
  if (D == 2) return b;
  csweep<D, N, 2>(b, a, mat, ncomp, NODES, NODES);
  __syncthreads();
  return a;
}

// Face tensors have D-1 directions of N points (NF total): sweep them all.
template <int D, int N>
__device__ __forceinline__ void face_sweep_all(double* data, double* tmp, const double* mat,
                                               int nblocks) {
  constexpr int NF = CShape<D, N>::NF;
  if (D == 2) {
    csweep<2, N, 0>(data, tmp, mat, nblocks, NF, NF);  // 1-D face: direction 0
    __syncthreads();
    for (int t = threadIdx.x; t < nblocks * NF; t += blockDim.x) data[t] = tmp[t];
    __syncthreads();
  } else {
    csweep<2, N, 0>(data, tmp, mat, nblocks, NF, NF);
    __syncthreads();
    csweep<2, N, 1>(tmp, data, mat, nblocks, NF, NF);
    __syncthreads();
  }
}

// Quadrature-space residual R (K u = B^T R) of one element; also leaves the
// Gauss values of u in uq.  Ends with a __syncthreads().
template <int D, int N>
__device__ void curved_residual(const AffineArgs& A, const CurvedArgs& G, double* sm,
                                long long e, double*& uq_out) {
  using S = CShape<D, N>;
  constexpr int C = S::C, NODES = S::NODES, NF = S::NF, TPB = S::TPB;
  double* us = sm + S::OFF_US;
  double* uqa = sm + S::OFF_UQ;
  double* tq = sm + S::OFF_TQ;
  double* R = sm + S::OFF_R;
  double* fl = sm + S::OFF_FL;
  double* nb = sm + S::OFF_NB;
  double* ftr = sm + S::OFF_FTR;
  double* ntr = sm + S::OFF_NTR;
  double* ftmp = sm + S::OFF_FTMP;
  const double* tab = sm + S::OFF_TAB;
  const double* tB = tab;
  const double* tBinv = tab + N * N;
  const double* tDco = tab + 2 * N * N;
  const double* tDcoT = tab + 3 * N * N;
  const int tid = threadIdx.x;
  for (int i = tid; i < 5 * N * N; i += TPB) sm[S::OFF_TAB + i] = G.ctab[i];
  for (int t = tid; t < C * NODES; t += TPB) us[t] = __ldg(A.u + e * C * NODES + t);
  const bool faces = (A.parts & PART_FACE) != 0;
  if (faces) {
    for (int t = tid; t < 2 * D * C * NF; t += TPB) {
      const int fn = t % NF;
      const int rest = t / NF;
      const int c = rest % C, f = rest / C;
      const int nbr = __ldg(A.nbr + e * 2 * D + f);
      WK_CHECK_NBR(A, nbr);
      double val = 0.0;
      if (nbr >= 0)
        val = __ldg(A.u + ((long long)nbr * C + c) * NODES +
                    face_to_node<N>(f >> 1, 1 - (f & 1), fn));
      else if (nbr <= -2)
        val = __ldg(A.ghost + ((long long)ghost_slot(nbr) * C + c) * NF + fn);
      nb[t] = val;
    }
  }
  __syncthreads();
  double* uq = csweep_all<D, N>(us, uqa, tq, tB, C);  // Gauss values
  double* spare = (uq == uqa) ? tq : uqa;
  uq_out = uq;
  if (faces) {
    // own face-node slices -> ftr, then GL->Gauss on both trace sets
    for (int t = tid; t < 2 * D * C * NF; t += TPB) {
      const int fn = t % NF;
      const int rest = t / NF;
      const int c = rest % C, f = rest / C;
      ftr[t] = us[c * NODES + face_to_node<N>(f >> 1, f & 1, fn)];
      ntr[t] = nb[t];
    }
    __syncthreads();
    face_sweep_all<D, N>(ftr, ftmp, tB, 2 * D * C);
    face_sweep_all<D, N>(ntr, ftmp, tB, 2 * D * C);
  }
  const double* mt = A.mat + e * kMatStride;
  const double ir = __ldg(mt + 0), c2r = __ldg(mt + 1), tau = __ldg(mt + 2);
  const double irt = __ldg(mt + 3);
  // pointwise: strong half -> R, weak fluxes -> fl
  const bool cell = (A.parts & PART_CELL) != 0;
  for (int pt = tid; pt < NODES; pt += TPB) {
    if (!cell) {
#pragma unroll
      for (int c = 0; c < C; ++c) R[c * NODES + pt] = 0.0;
      continue;
    }
    double Gm[D][D];
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
      for (int i = 0; i < D; ++i)
        Gm[m][i] = __ldg(G.inv_jac + ((e * D + m) * D + i) * (long long)NODES + pt);
    const double jw = __ldg(G.jxw + e * NODES + pt);
    double grad[D][C];
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int sm_ = m == 0 ? 1 : (m == 1 ? N : N * N);
      const int im = (pt / sm_) % N;
      const int base = pt - im * sm_;
      const double* row = tDco + im * N;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) s = fma(row[j], uq[c * NODES + base + j * sm_], s);
        grad[m][c] = s;
      }
    }
    const double hv = 0.5 * jw * ir, hp = 0.5 * jw * c2r;
    double sv[D], spp = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) sv[i] = 0.0;
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
      for (int i = 0; i < D; ++i) {
        sv[i] = fma(Gm[m][i], grad[m][D], sv[i]);
        spp = fma(Gm[m][i], grad[m][i], spp);
      }
#pragma unroll
    for (int i = 0; i < D; ++i) R[i * NODES + pt] = hv * sv[i];
    R[D * NODES + pt] = hp * spp;
    const double pq = uq[D * NODES + pt];
#pragma unroll
    for (int m = 0; m < D; ++m) {
      double vg = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        fl[(m * C + i) * NODES + pt] = -hv * Gm[m][i] * pq;
        vg = fma(Gm[m][i], uq[i * NODES + pt], vg);
      }
      fl[(m * C + D) * NODES + pt] = -hp * vg;
    }
  }
  if (faces) {
    // face integrand at the face Gauss points (operator.py:224-240), into ntr
    for (int t = tid; t < 2 * D * NF; t += TPB) {
      const int fn = t % NF, f = t / NF;
      const int nbr = __ldg(A.nbr + e * 2 * D + f);
      double own[C], oth[C];
#pragma unroll
      for (int c = 0; c < C; ++c) own[c] = ftr[(f * C + c) * NF + fn];
      if (nbr == -1) {
#pragma unroll
        for (int c = 0; c < D; ++c) oth[c] = own[c];
        oth[D] = -own[D];
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) oth[c] = ntr[(f * C + c) * NF + fn];
      }
      double nrm[D], vn_o = 0.0, vn_x = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        nrm[i] = __ldg(G.fnormal[f] + (e * D + i) * NF + fn);
        vn_o = fma(nrm[i], own[i], vn_o);
        vn_x = fma(nrm[i], oth[i], vn_x);
      }
      double pv = 0.5 * ir * oth[D];
      double pp = 0.5 * c2r * vn_x;
      if (A.stab) {
        pv += 0.5 * irt * (vn_o - vn_x);
        pp += 0.5 * c2r * tau * (own[D] - oth[D]);
      }
      const double fj = __ldg(G.fjxw[f] + e * NF + fn);
#pragma unroll
      for (int i = 0; i < D; ++i) ntr[(f * C + i) * NF + fn] = pv * nrm[i] * fj;
      ntr[(f * C + D) * NF + fn] = pp * fj;
    }
  }
  __syncthreads();
  // weak half (D_co^T along m) and face lifts (GL-endpoint rows of B^{-1})
  for (int t = tid; t < C * NODES; t += TPB) {
    const int c = t / NODES, pt = t - c * NODES;
    double acc = R[t];
    int sm_ = 1;
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int im = (pt / sm_) % N;
      const int base = pt - im * sm_;
      if (cell) {
        const double* src = fl + (m * C + c) * NODES + base;
        const double* row = tDcoT + im * N;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) s = fma(row[j], src[j * sm_], s);
        acc += s;
      }
      if (faces) {
        const int fn = node_to_face<N>(m, pt);
        const double l0 = tBinv[0 * N + im], l1 = tBinv[(N - 1) * N + im];
        acc = fma(l0, ntr[((2 * m) * C + c) * NF + fn],
                  fma(l1, ntr[((2 * m + 1) * C + c) * NF + fn], acc));
      }
      sm_ *= N;
    }
    spare[t] = acc;  // final residual in `spare`
  }
  __syncthreads();
  for (int t = tid; t < C * NODES; t += TPB) R[t] = spare[t];
  __syncthreads();
}

template <int D, int N, int MODE>
__global__ void __launch_bounds__(CShape<D, N>::TPB)
curved_op_kernel(AffineArgs A, CurvedArgs G) {
  using S = CShape<D, N>;
  constexpr int C = S::C, NODES = S::NODES, TPB = S::TPB;
  extern __shared__ double sm[];
  const long long e = A.e_begin + blockIdx.x;
  double* uq;
  curved_residual<D, N>(A, G, sm, e, uq);
  double* R = sm + S::OFF_R;
  double* a = sm + S::OFF_UQ;
  double* b = sm + S::OFF_TQ;
  const double* tab = sm + S::OFF_TAB;
  const double* us = sm + S::OFF_US;
  double* res;
  if (MODE == OUT_K) {
    res = csweep_all<D, N>(R, a, b, tab + 4 * N * N, C);  // B^T
  } else {
    for (int t = threadIdx.x; t < C * NODES; t += TPB)
      R[t] /= __ldg(G.jxw + e * NODES + (t % NODES));
    __syncthreads();
    res = csweep_all<D, N>(R, a, b, tab + N * N, C);      // B^{-1}
  }
  for (int t = threadIdx.x; t < C * NODES; t += TPB) {
    const long long idx = e * C * NODES + t;
    const double v = res[t];
    if (MODE == OUT_K || MODE == OUT_MINVK) {
      A.out[idx] = v;
    } else if (MODE == OUT_RHS) {
      A.out[idx] = -v;
    } else if (MODE == OUT_LSRK) {
      const double f = -v * A.dt;
      const double rr = A.a == 0.0 ? f : fma(A.a, A.r[idx], f);
      A.r[idx] = rr;
      A.u_out[idx] = fma(A.b, rr, us[t]);
    } else if (MODE == OUT_ADERB) {
      A.out[idx] = A.v[idx] - v;
    }
  }
}

// ---- curved TCK ------------------------------------------------------------
// S at degree NN-1 with the per-point metric of that degree (operator.py:286-306)
template <int D, int N, int NN>
__device__ __forceinline__ void ctck_apply_S_ct(const double* cur, double* nxt,
                                                const double* dm, const double* ij,
                                                double ir, double c2r, long long e) {
  constexpr int C = D + 1, NODES = CShape<D, N>::NODES, TPB = CShape<D, N>::TPB;
  constexpr int nodes = D == 3 ? NN * NN * NN : NN * NN;
  for (int pt = threadIdx.x; pt < nodes; pt += TPB) {
    double grad[D][C];
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int sm_ = m == 0 ? 1 : (m == 1 ? NN : NN * NN);
      const int im = (pt / sm_) % NN;
      const int base = pt - im * sm_;
      const double* row = dm + im * NN;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NN; ++j) s = fma(row[j], cur[c * NODES + base + j * sm_], s);
        grad[m][c] = s;
      }
    }
    double sv[D], sp = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) sv[i] = 0.0;
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double gmi = __ldg(ij + ((e * D + m) * D + i) * (long long)nodes + pt);
        sv[i] = fma(gmi, grad[m][D], sv[i]);
        sp = fma(gmi, grad[m][i], sp);
      }
#pragma unroll
    for (int i = 0; i < D; ++i) nxt[i * NODES + pt] = ir * sv[i];
    nxt[D * NODES + pt] = c2r * sp;
  }
  __syncthreads();
}

template <int D, int N>
__device__ __forceinline__ void ctck_apply_S(const TckArgs& T, const CurvedArgs& G,
                                             double*& cur, double*& nxt, const double* dm,
                                             int n, long long e) {
  const double ir = __ldg(T.op.mat + e * kMatStride + 0);
  const double c2r = __ldg(T.op.mat + e * kMatStride + 1);
  const double* ij = G.invjac_deg[n - 1];
  switch (n) {
#define WK_CS(k)                                                                       \
  case k:                                                                              \
    if constexpr (k <= N) ctck_apply_S_ct<D, N, k>(cur, nxt, dm, ij, ir, c2r, e);       \
    break;
    WK_CS(1) WK_CS(2) WK_CS(3) WK_CS(4) WK_CS(5) WK_CS(6) WK_CS(7) WK_CS(8)
#undef WK_CS
  }
  double* t = cur; cur = nxt; nxt = t;
}

template <int D, int N>
struct CTckSmem {
  using S = CShape<D, N>;
  static size_t bytes(int acc_len, int tab_len) {
    return sizeof(double) * (size_t)(S::TOTAL + acc_len + tab_len);
  }
};

// Curved ADER kernel A (one element per CTA): (hdg) W = M^{-1}K U at the
// Gauss points, V = U - dt W, y = TCK_shift(W); (plain) y = TCK(U).
template <int D, int N, bool HDG>
__global__ void __launch_bounds__(CShape<D, N>::TPB)
curved_ader_a_kernel(const __grid_constant__ TckArgs T, const __grid_constant__ CurvedArgs G) {
  using S = CShape<D, N>;
  constexpr int C = S::C, NODES = S::NODES, TPB = S::TPB;
  extern __shared__ double sm[];
  double* acc = sm + S::TOTAL;
  double* ttab = acc + T.acc_len;
  const long long e = T.op.e_begin + blockIdx.x;
  const int tid = threadIdx.x;
  for (int i = tid; i < T.tab_len; i += TPB) ttab[i] = T.tck_tab[i];
  double* cur;
  double* nxt;
  const double* tab = sm + S::OFF_TAB;
  if (HDG) {
    double* uq;
    const AffineArgs op = T.op;
    curved_residual<D, N>(op, G, sm, e, uq);
    double* R = sm + S::OFF_R;
    for (int t = tid; t < C * NODES; t += TPB) R[t] /= __ldg(G.jxw + e * NODES + (t % NODES));
    __syncthreads();
    // W (GL) for V = U - dt W; R keeps W at the Gauss points
    double* w = csweep_all<D, N>(R, sm + S::OFF_UQ, sm + S::OFF_TQ, tab + N * N, C);
    const double* us = sm + S::OFF_US;
    for (int t = tid; t < C * NODES; t += TPB)
      T.v_out[e * C * NODES + t] = us[t] - T.dt * w[t];
    __syncthreads();
    cur = R;
    nxt = sm + S::OFF_UQ;
  } else {
    double* us = sm + S::OFF_US;
    for (int i = tid; i < 5 * N * N; i += TPB) sm[S::OFF_TAB + i] = G.ctab[i];
    for (int t = tid; t < C * NODES; t += TPB) us[t] = __ldg(T.op.u + e * C * NODES + t);
    __syncthreads();
    cur = csweep_all<D, N>(us, sm + S::OFF_UQ, sm + S::OFF_TQ, tab, C);  // Gauss values
    nxt = (cur == sm + S::OFF_UQ) ? sm + S::OFF_TQ : sm + S::OFF_UQ;
  }
  for (int op = 0; op < T.nops; ++op) {
    const int code = __ldg(T.prog + 4 * op + 0);
    const int a0 = __ldg(T.prog + 4 * op + 1);
    const int a1 = __ldg(T.prog + 4 * op + 2);
    const int a2 = __ldg(T.prog + 4 * op + 3);
    if (code == TCK_S) {
      ctck_apply_S<D, N>(T, G, cur, nxt, ttab + a1, a0, e);
    } else if (code == TCK_RESIZE) {
      gader_resize<D, N, TPB>(cur, nxt, ttab + a2, a0, a1, tid);
    } else {
      const double w = T.w[op];
      const int nn = npow<D>(a1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double* slot = acc + a0 + c * nn;
        double* cv = cur + c * NODES;
        if (code == TCK_ACC_SET) {
          for (int pt = tid; pt < nn; pt += TPB) slot[pt] = w * cv[pt];
        } else if (code == TCK_ACC_ADD) {
          for (int pt = tid; pt < nn; pt += TPB) slot[pt] = slot[pt] + w * cv[pt];
        } else {
          for (int pt = tid; pt < nn; pt += TPB) cv[pt] = slot[pt];
        }
      }
      __syncthreads();
    }
  }
  // acc_k (Gauss values) -> y
  double* a = cur;
  double* b = nxt;
  if (G.y_mode == 0) {
    double* y = csweep_all<D, N>(acc, a, b, tab + N * N, C);  // B^{-1}
    for (int t = tid; t < C * NODES; t += TPB) T.y[e * C * NODES + t] = y[t];
  } else {
    for (int t = tid; t < C * NODES; t += TPB)
      acc[t] *= __ldg(G.jxw + e * NODES + (t % NODES));
    __syncthreads();
    double* y = csweep_all<D, N>(acc, a, b, tab + 4 * N * N, C);  // B^T
    for (int t = tid; t < C * NODES; t += TPB) T.y[e * C * NODES + t] = y[t];
  }
}

}  // namespace wk
