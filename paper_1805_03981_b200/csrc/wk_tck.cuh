// Element-local Taylor-Cauchy-Kowalevski (TCK) kernel for ADER on general
// (sheared / multi-class) affine elements.
//
// Reference: tck_evaluate (stepping.py:215-262) with apply_local_S /
// resize_values / to_gauss_values / from_gauss_weighted (operator.py:276-325)
// and reduction_schedule (kernels.py:286-302).  The host compiles that loop
// -- including the degree-0 break, the shift re-indexing and the accumulator
// chain-up -- into a short op program (wk_abi.cu: build_tck_program) that this
// kernel interprets with all data resident in shared memory.
//
// Basis: on affine cells every step of the Taylor loop is an exact polynomial
// operation, so the full-degree field stays in the GL basis (S uses the GL
// collocation derivative) while reduced degrees use Gauss collocation as in the
// reference.  This removes the reference's GL->Gauss entry and Gauss->GL exit
// sweeps; M^{-1} T = B^{-1} acc_k (operator.py:250-258, 279-284) is then simply
// acc_k, which the kernel writes as y.
#pragma once
#include "wk_affine.cuh"

namespace wk {

enum TckOp : int { TCK_S = 0, TCK_RESIZE = 1, TCK_ACC_SET = 2, TCK_ACC_ADD = 3, TCK_LOAD = 4 };

constexpr int kTckOps = 96;  // longest op program (k = 8, every_step, no shift) is < 64

struct TckArgs {
  AffineArgs op;          // operator inputs (u = U), geometry, material
  double* y;              // output: M^{-1} T  (GL coefficients)
  double* v_out;          // ADER-HDG: V = U - dt W  (null for plain ADER)
  const int* prog;        // (nops, 4)
  // per-op weights (Taylor weight of this dt, or 1) BY VALUE: a launch --
  // and a CUDA graph that captured it -- carries its own dt's weights
  double w[kTckOps];
  const double* tck_tab;  // matrices referenced by the program
  int nops;
  int tab_len;            // doubles in tck_tab
  int acc_len;            // doubles per element in the accumulator block
  double dt;
};

template <int D>
__device__ __forceinline__ int npow(int n) { return D == 3 ? n * n * n : n * n; }

// Dynamic smem carve-up for ader_a_kernel (doubles).
template <int D, int N, bool CART>
struct TckSmem {
  using S = Shape<D, N>;
  static constexpr int OPREG = AffineSmem<D, N, CART>::US + AffineSmem<D, N, CART>::NB +
                               AffineSmem<D, N, CART>::WS;
  static constexpr int TCKREG = 2 * S::EPB * S::C * S::NODES + S::EPB * D * S::NODES;
  static constexpr int R1 = OPREG > TCKREG ? OPREG : TCKREG;
  static constexpr int OPTAB = N * N + 2 * N;
  __host__ __device__ static size_t bytes(int acc_len, int tab_len) {
    return sizeof(double) * (size_t)(R1 + OPTAB + S::EPB * acc_len + tab_len);
  }
};

// Pointwise S on collocated values at n points per direction (operator.py:286-306):
//   out_i = rho^{-1} sum_m G[m,i] d_m p,   out_p = c^2 rho sum_m d_m (sum_i G[m,i] v_i)
template <int D, int N, bool CART>
__device__ __forceinline__ void tck_apply_S(const TckArgs& A, double*& cur, double*& nxt,
                                            double* wb, const double* dm, int n,
                                            long long e0, int nel) {
  using S = Shape<D, N>;
  constexpr int C = S::C, NODES = S::NODES, EPB = S::EPB, TPB = S::TPB;
  const int nodes = npow<D>(n);
  const int tid = threadIdx.x;
  if (!CART) {
    for (int t = tid; t < EPB * nodes; t += TPB) {
      const int el = t / nodes, pt = t - el * nodes;
      if (el >= nel) continue;
      const int cls = A.op.geo_class ? __ldg(A.op.geo_class + e0 + el) : 0;
      const double* g = A.op.geo + (long long)cls * GeoLayout<D>::STRIDE;
#pragma unroll
      for (int m = 0; m < D; ++m) {
        double w = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) w = fma(__ldg(g + m * D + i), cur[(el * C + i) * NODES + pt], w);
        wb[(el * D + m) * NODES + pt] = w;
      }
    }
    __syncthreads();
  }
  for (int t = tid; t < EPB * nodes; t += TPB) {
    const int el = t / nodes, pt = t - el * nodes;
    if (el >= nel) continue;
    const long long e = e0 + el;
    const int cls = A.op.geo_class ? __ldg(A.op.geo_class + e) : 0;
    const double* g = A.op.geo + (long long)cls * GeoLayout<D>::STRIDE;
    const double ir = __ldg(A.op.mat + e * kMatStride + 0);
    const double c2r = __ldg(A.op.mat + e * kMatStride + 1);
    double res[C];
#pragma unroll
    for (int c = 0; c < C; ++c) res[c] = 0.0;
    const double* up = cur + (el * C + D) * NODES;
    int sm = 1;
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int im = (pt / sm) % n;
      const int base = pt - im * sm;
      const double* row = dm + im * n;
      const double* wl = CART ? cur + (el * C + m) * NODES : wb + (el * D + m) * NODES;
      double dp = 0.0, dw = 0.0;
      for (int j = 0; j < n; ++j) {
        dp = fma(row[j], up[base + j * sm], dp);
        dw = fma(row[j], wl[base + j * sm], dw);
      }
      if (CART) {
        const double gmm = __ldg(g + m * D + m);
        res[m] = fma(ir * gmm, dp, res[m]);
        res[D] = fma(c2r * gmm, dw, res[D]);
      } else {
#pragma unroll
        for (int i = 0; i < D; ++i) res[i] = fma(ir * __ldg(g + m * D + i), dp, res[i]);
        res[D] = fma(c2r, dw, res[D]);
      }
      sm *= n;
    }
#pragma unroll
    for (int c = 0; c < C; ++c) nxt[(el * C + c) * NODES + pt] = res[c];
  }
  __syncthreads();
  double* t = cur; cur = nxt; nxt = t;
}

// Resize every direction nf -> nt with an (nt x nf) matrix (operator.py:308-325).
template <int D, int N>
__device__ __forceinline__ void tck_resize(double*& cur, double*& nxt, const double* mat,
                                           int nf, int nt, int nel) {
  using S = Shape<D, N>;
  constexpr int C = S::C, NODES = S::NODES, EPB = S::EPB, TPB = S::TPB;
  const int tid = threadIdx.x;
  for (int m = 0; m < D; ++m) {
    int ein[3] = {1, 1, 1}, eout[3] = {1, 1, 1};
    for (int q = 0; q < D; ++q) {
      ein[q] = q < m ? nt : nf;
      eout[q] = q <= m ? nt : nf;
    }
    const int tot = eout[0] * eout[1] * eout[2];
    const int sin_m = m == 0 ? 1 : (m == 1 ? ein[0] : ein[0] * ein[1]);
    for (int t = tid; t < EPB * C * tot; t += TPB) {
      const int ec = t / tot, pt = t - ec * tot;
      const int el = ec / C;
      if (el >= nel) continue;
      const int i0 = pt % eout[0], i1 = (pt / eout[0]) % eout[1], i2 = pt / (eout[0] * eout[1]);
      const int idx[3] = {i0, i1, i2};
      // input linear index with idx[m] replaced by j
      int lin = 0, stride = 1;
      for (int q = 0; q < D; ++q) {
        if (q != m) lin += idx[q] * stride;
        stride *= ein[q];
      }
      const double* src = cur + ec * NODES + lin;
      const double* row = mat + idx[m] * nf;
      double s = 0.0;
      for (int j = 0; j < nf; ++j) s = fma(row[j], src[j * sin_m], s);
      nxt[ec * NODES + pt] = s;
    }
    __syncthreads();
    double* tt = cur; cur = nxt; nxt = tt;
  }
}

// ADER kernel A on general affine cells: y = M^{-1} TCK(u) (stepping.py:215-262).
// ADER-HDG on these meshes composes it with the stage kernel (wk_abi.cu
// run_ader_a): W = M^{-1} K U, V = U - dt W, then this kernel on W with the
// shift.  (A fused HDG variant of this kernel, with the operator's stage
// functions inlined in front of the Taylor loop, faulted at -O3 for 3-D
// n >= 7 on non-Cartesian cells and ran clean at -Xptxas -O1, with no spills
// and only explicit global / shared accesses in its SASS; it was removed,
// DESIGN.md §8.)
template <int D, int N, bool CART>
__global__ void __launch_bounds__(Shape<D, N>::TPB)
ader_a_kernel(const __grid_constant__ TckArgs A) {
  using S = Shape<D, N>;
  using TS = TckSmem<D, N, CART>;
  constexpr int C = S::C, NODES = S::NODES, EPB = S::EPB, TPB = S::TPB;
  extern __shared__ double smem[];
  double* r1 = smem;
  double* optab = r1 + TS::R1;
  double* acc = optab + TS::OPTAB;
  double* ttab = acc + EPB * A.acc_len;
  const int tid = threadIdx.x;
  const int el = tid / NODES;
  const int node = tid - el * NODES;
  const long long e0 = A.op.e_begin + (long long)blockIdx.x * EPB;
  const long long e = e0 + el;
  const long long e_end = A.op.e_begin + A.op.E;
  const bool active = el < EPB && e < e_end;
  const int nel = (int)((e_end - e0) < EPB ? (e_end - e0) : EPB);
  WK_CHECK_SMEM(TS::bytes(A.acc_len, A.tab_len));
  for (int i = tid; i < A.tab_len; i += TPB) ttab[i] = A.tck_tab[i];

  double* cur = r1;
  double* nxt = r1 + EPB * C * NODES;
  double* wb = nxt + EPB * C * NODES;
  if (active) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      cur[(el * C + c) * NODES + node] = __ldg(A.op.u + (e * C + c) * NODES + node);
  }
  __syncthreads();

  int n = N;  // current points per direction
  for (int op = 0; op < A.nops; ++op) {
    const int code = __ldg(A.prog + 4 * op + 0);
    const int a0 = __ldg(A.prog + 4 * op + 1);
    const int a1 = __ldg(A.prog + 4 * op + 2);
    const int a2 = __ldg(A.prog + 4 * op + 3);
    if (code == TCK_S) {
      tck_apply_S<D, N, CART>(A, cur, nxt, wb, ttab + a1, a0, e0, nel);
    } else if (code == TCK_RESIZE) {
      tck_resize<D, N>(cur, nxt, ttab + a2, a0, a1, nel);
      n = a1;
    } else {
      const double w = A.w[op];
      const int nn = npow<D>(a1);
      for (int t = tid; t < EPB * C * nn; t += TPB) {
        const int ec = t / nn, pt = t - ec * nn;
        const int el2 = ec / C, c = ec - el2 * C;
        if (el2 >= nel) continue;
        double* slot = acc + el2 * A.acc_len + a0 + c * nn + pt;
        double* cv = cur + ec * NODES + pt;
        if (code == TCK_ACC_SET) *slot = w * *cv;
        else if (code == TCK_ACC_ADD) *slot = *slot + w * *cv;
        else *cv = *slot;  // TCK_LOAD
      }
      if (code == TCK_LOAD) n = a1;
      __syncthreads();
    }
  }
  (void)n;
  // slot 0 holds acc_k in the GL basis = M^{-1} T
  if (active) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      A.y[(e * C + c) * NODES + node] = acc[el * A.acc_len + c * NODES + node];
  }
}

}  // namespace wk
