// Fused FP64 kernels for affine (constant-Jacobian) hexahedral/quadrilateral
// elements.
//
// Formulation (proven identical to the reference in
// tests/test_formulation.py): on an affine cell J^{-1} and det J are constant
// and every integral the reference evaluates by Gauss quadrature
// (operator.py:149-246) is exact, so M^{-1} K collapses to 1-D operators on
// the GL coefficients:
//
//   (M^{-1} K u)_v_i = rho^{-1} sum_m G[m,i] A_m p           (cell, split form)
//   (M^{-1} K u)_p   = c^2 rho sum_m A_m (sum_i G[m,i] v_i)
//                      + sum_{m,s} fscale_{m,s} L_s(xi_m) (x) F_{m,s}   (faces)
//
// with A = 1/2 M1^{-1} (B^T W D_gl - D_gl^T W B) (the split strong/weak cell
// form of operator.py:157-187 in one n x n matrix), L_s = M1^{-1} e_{end(s)}
// the lifted face test function, and F_{m,s} the reference's face integrand
// u_hat - F_n(own)/2 (operator.py:224-239) evaluated pointwise on the GL face
// nodes.  Per element: 2d sweeps of an n x n matrix plus 2d rank-1 lifts --
// against 27 sweeps x 4 components plus 6 mass sweeps in the reference.
#pragma once
#include "wk_common.cuh"

namespace wk {

struct AffineArgs {
  const double* u;        // operator input state (E, C, NODES)
  double* out;            // OUT_MINVK / OUT_RHS / OUT_ADERB output
  double* r;              // OUT_LSRK register (in/out)
  double* u_out;          // OUT_LSRK new state (must not alias u)
  const double* v;        // OUT_ADERB: V (may alias out)
  const int* nbr;         // (E, d, 2) int32
  const double* ghost;    // (G, C, NF) halo face slices or null
  const double* geo;      // (n_classes, GeoLayout::STRIDE)
  const int* geo_class;   // (E,) or null -> class 0
  const double* mat;      // (E, kMatStride)
  const double* tab;      // A (N*N), L0 (N), L1 (N)
  long long E;            // elements in this launch's range
  long long e_begin;      // first element of the range (element offset)
  double a, b, dt;        // LSRK coefficients
  int parts;              // Parts bitmask
  int stab;               // stabilization on/off (FluxParams.stabilization)
  int has_ghost;          // any neighbour code <= -2 (multi-GPU halo slots)
  int r_dead;             // OUT_LSRK: r is dead after this stage, do not store it
  unsigned* sched;        // persistent kernels' tile queue {claim, done}, zero between launches
  int l2pf;               // persistent kernels: bulk-prefetch tiles two ahead into L2
  int grid_hold;          // persistent kernels: SMs' worth of CTA slots left free
  // persistent kernels: structured traversal (wk_set_tile_order): the range
  // is n_slow x n_blocks chunks of tmap_ch elements (slow to fast), visited
  // block-major, so both slow-axis neighbours of a chunk are streamed just
  // before / after it (their faces hit in L2).  tmap_ch = 0: mesh order.
  unsigned tmap_ch, tmap_ns, tmap_nb;
  // ceil(2^32 / tmap_ch), ceil(2^32 / tmap_ns): the map's two divisions as
  // one umulhi each (exact while E * tmap_ch < 2^32, checked on the host)
  unsigned tmap_ch_m, tmap_ns_m;
  long long e_total;      // elements of the whole mesh (checked build: neighbour bounds)
  long long n_ghost;      // ghost face slots (checked build)
  // the same 1-D tables by value: kernel parameters live in the constant
  // bank, so the pencil kernels' DFMAs read them as c[][] operands without
  // any load instruction
  double cA[kMaxN * kMaxN];
  double cL0[kMaxN], cL1[kMaxN];
};

// First element of tile t (tiles of EPG elements, in traversal order).
template <int EPG>
__device__ __forceinline__ long long tile_elem(const AffineArgs& a, long long t) {
  if (a.tmap_ch == 0) return a.e_begin + t * EPG;
  const unsigned lin = (unsigned)t * (unsigned)EPG;   // host: E < 2^32
  const unsigned c = a.tmap_ch > 1 ? __umulhi(lin, a.tmap_ch_m) : lin, r = lin - c * a.tmap_ch;
  const unsigned b = a.tmap_ns > 1 ? __umulhi(c, a.tmap_ns_m) : c, sl = c - b * a.tmap_ns;
  const long long e = a.e_begin + (long long)(sl * a.tmap_nb + b) * a.tmap_ch + r;
  WK_ASSERT(e >= a.e_begin && e < a.e_begin + a.E);
  return e;
}

template <int N>
__device__ __forceinline__ constexpr int ipow(int m) {
  return m == 0 ? 1 : (m == 1 ? N : N * N);
}

// node index of face (m, side) node fn (constant divisors in every branch,
// so a runtime m never reaches the integer-division subroutine)
template <int N>
__device__ __forceinline__ int face_to_node(int m, int side, int fn) {
  if (m == 0) return side * (N - 1) + fn * N;
  if (m == 1) return fn % N + side * (N - 1) * N + (fn / N) * N * N;
  return fn + side * (N - 1) * N * N;
}

// first node (i_m = 0) of the pencil along m through face node fn
template <int N>
__device__ __forceinline__ int pencil_base(int m, int fn) {
  if (m == 0) return fn * N;
  if (m == 1) return fn % N + (fn / N) * N * N;
  return fn;
}

// face-node index of a volume node for direction m
template <int N>
__device__ __forceinline__ int node_to_face(int m, int node) {
  if (m == 0) return node / N;
  if (m == 1) return node % N + (node / (N * N)) * N;
  return node % (N * N);
}

// Dynamic shared-memory footprint of affine_op_kernel (doubles).
template <int D, int N, bool CART>
struct AffineSmem {
  using S = Shape<D, N>;
  static constexpr int US = S::EPB * S::C * S::NODES;
  static constexpr int NB = S::EPB * 2 * D * S::C * S::NF;
  static constexpr int WS = CART ? 0 : S::EPB * D * S::NODES;
  static constexpr int TAB = N * N + 2 * N;
  static constexpr size_t BYTES = sizeof(double) * (US + NB + WS + TAB);
};

// Stage 1 of every affine operator kernel: own state -> smem/registers,
// neighbour face-node slices -> smem, face integrands (in place), and the
// non-Cartesian flux combinations w_m = sum_i G[m,i] v_i.
template <int D, int N, bool CART>
__device__ __forceinline__ void affine_stage_inputs(
    const AffineArgs& args, double* us, double* nb, double* ws, double* tabs,
    double (&uv)[D + 1], int el, int node, long long e, bool active) {
  using S = Shape<D, N>;
  constexpr int C = S::C, NODES = S::NODES, NF = S::NF, EPB = S::EPB, TPB = S::TPB;
  using GL_ = GeoLayout<D>;
  const int tid = threadIdx.x;
  for (int i = tid; i < N * N + 2 * N; i += TPB) tabs[i] = args.tab[i];
  if (active) {
    const double* src = args.u + (e * C) * NODES + node;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      uv[c] = __ldg(src + c * NODES);
      us[(el * C + c) * NODES + node] = uv[c];
    }
  }
  const long long e0 = args.e_begin + (long long)blockIdx.x * EPB;
  if (args.parts & PART_FACE) {
    constexpr int TOT = EPB * 2 * D * C * NF;
    for (int t = tid; t < TOT; t += TPB) {
      const int fn = t % NF;
      int rest = t / NF;
      const int c = rest % C;
      rest /= C;
      const int f = rest % (2 * D);
      const int el2 = rest / (2 * D);
      const long long e2 = e0 + el2;
      if (e2 >= args.e_begin + args.E) continue;
      const int nbr = __ldg(args.nbr + e2 * 2 * D + f);
      double val = 0.0;
WK_CHECK_NBR(args, nbr);
      if (nbr >= 0) {
        val = __ldg(args.u + ((long long)nbr * C + c) * NODES +
                    face_to_node<N>(f >> 1, 1 - (f & 1), fn));
      } else if (nbr <= -2) {
        val = __ldg(args.ghost + ((long long)ghost_slot(nbr) * C + c) * NF + fn);
      }
      nb[((el2 * 2 * D + f) * C + c) * NF + fn] = val;
    }
  }
  __syncthreads();
  if (args.parts & PART_FACE) {
#pragma unroll
    for (int f = 0; f < 2 * D; ++f) {
      const int m = f >> 1, s = f & 1;
      for (int t = tid; t < EPB * NF; t += TPB) {
        const int el2 = t / NF, fn = t - (t / NF) * NF;
        const long long e2 = e0 + el2;
        if (e2 >= args.e_begin + args.E) continue;
        const int nbr = __ldg(args.nbr + e2 * 2 * D + f);
        const int cls = args.geo_class ? __ldg(args.geo_class + e2) : 0;
        const double* g = args.geo + (long long)cls * GL_::STRIDE;
        const double* mt = args.mat + e2 * kMatStride;
        const double ir = __ldg(mt + 0), c2r = __ldg(mt + 1), tau = __ldg(mt + 2);
        const double irt = __ldg(mt + 3);
        const int on = face_to_node<N>(m, s, fn);
        double own[C], oth[C];
        double* slot = nb + ((el2 * 2 * D + f) * C) * NF + fn;
#pragma unroll
        for (int c = 0; c < C; ++c) own[c] = us[(el2 * C + c) * NODES + on];
        if (nbr == -1) {  // sound-soft mirror: velocity kept, pressure negated
#pragma unroll
          for (int c = 0; c < D; ++c) oth[c] = own[c];
          oth[D] = -own[D];
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) oth[c] = slot[c * NF];
        }
        double nrm[D];
        double vn_o = 0.0, vn_x = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          nrm[i] = __ldg(g + GL_::NORMAL + (m * 2 + s) * D + i);
          vn_o = fma(nrm[i], own[i], vn_o);
          vn_x = fma(nrm[i], oth[i], vn_x);
        }
        double pv = 0.5 * ir * oth[D];
        double pp = 0.5 * c2r * vn_x;
        if (args.stab) {
          pv += 0.5 * irt * (vn_o - vn_x);
          pp += 0.5 * c2r * tau * (own[D] - oth[D]);
        }
        const double fs = __ldg(g + GL_::FSCALE + m * 2 + s);
#pragma unroll
        for (int i = 0; i < D; ++i) slot[i * NF] = pv * nrm[i] * fs;
        slot[D * NF] = pp * fs;
      }
    }
  }
  if (!CART && active && (args.parts & PART_CELL)) {
    const int cls = args.geo_class ? __ldg(args.geo_class + e) : 0;
    const double* g = args.geo + (long long)cls * GL_::STRIDE;
#pragma unroll
    for (int m = 0; m < D; ++m) {
      double w = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) w = fma(__ldg(g + m * D + i), uv[i], w);
      ws[(el * D + m) * NODES + node] = w;
    }
  }
  __syncthreads();
}

// Stage 2: res = (M^{-1} K u) at this thread's node.
template <int D, int N, bool CART>
__device__ __forceinline__ void affine_node_result(
    const AffineArgs& args, const double* us, const double* nb, const double* ws,
    const double* tabs, int el, int node, long long e, double (&res)[D + 1]) {
  using S = Shape<D, N>;
  constexpr int C = S::C, NODES = S::NODES, NF = S::NF;
#pragma unroll
  for (int c = 0; c < C; ++c) res[c] = 0.0;
  const double* sA = tabs;
  const double* sL0 = tabs + N * N;
  const double* sL1 = sL0 + N;
  if (args.parts & PART_CELL) {
    const int cls = args.geo_class ? __ldg(args.geo_class + e) : 0;
    const double* g = args.geo + (long long)cls * GeoLayout<D>::STRIDE;
    const double* mt = args.mat + e * kMatStride;
    const double ir = __ldg(mt + 0), c2r = __ldg(mt + 1);
    const double* up = us + (el * C + D) * NODES;
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
      const int im = (node / sm) % N;
      const int base = node - im * sm;
      const double* arow = sA + im * N;
      const double* wl = CART ? us + (el * C + m) * NODES : ws + (el * D + m) * NODES;
      double dp = 0.0, dw = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double a = arow[j];
        dp = fma(a, up[base + j * sm], dp);
        dw = fma(a, wl[base + j * sm], dw);
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
    }
  }
  if (args.parts & PART_FACE) {
#pragma unroll
    for (int m = 0; m < D; ++m) {
      const int sm = m == 0 ? 1 : (m == 1 ? N : N * N);
      const int im = (node / sm) % N;
      const int fn = node_to_face<N>(m, node);
      const double l0 = sL0[im], l1 = sL1[im];
      const double* f0 = nb + ((el * 2 * D + 2 * m) * C) * NF + fn;
      const double* f1 = f0 + C * NF;
#pragma unroll
      for (int c = 0; c < C; ++c) res[c] = fma(l0, f0[c * NF], fma(l1, f1[c * NF], res[c]));
    }
  }
}

template <int D, int N, bool CART, int MODE>
__global__ void __launch_bounds__(Shape<D, N>::TPB)
affine_op_kernel(AffineArgs args) {
  using S = Shape<D, N>;
  using SM = AffineSmem<D, N, CART>;
  constexpr int C = S::C, NODES = S::NODES, EPB = S::EPB;
  extern __shared__ double smem[];
  double* us = smem;
  double* nb = us + SM::US;
  double* ws = nb + SM::NB;
  double* tabs = ws + SM::WS;
  const int el = threadIdx.x / NODES;
  const int node = threadIdx.x - el * NODES;
  const long long e = args.e_begin + (long long)blockIdx.x * EPB + el;
  const bool active = el < EPB && e < args.e_begin + args.E;
  double uv[C];
#pragma unroll
  for (int c = 0; c < C; ++c) uv[c] = 0.0;
  affine_stage_inputs<D, N, CART>(args, us, nb, ws, tabs, uv, el, node, e, active);
  if (!active) return;
  double res[C];
  affine_node_result<D, N, CART>(args, us, nb, ws, tabs, el, node, e, res);
  const long long base = (e * C) * NODES + node;
  if (MODE == OUT_MINVK) {
#pragma unroll
    for (int c = 0; c < C; ++c) args.out[base + c * NODES] = res[c];
  } else if (MODE == OUT_RHS) {
#pragma unroll
    for (int c = 0; c < C; ++c) args.out[base + c * NODES] = -res[c];
  } else if (MODE == OUT_LSRK) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const long long idx = base + c * NODES;
      const double f = -res[c] * args.dt;
      const double rr = args.a == 0.0 ? f : fma(args.a, args.r[idx], f);
      args.r[idx] = rr;
      args.u_out[idx] = fma(args.b, rr, uv[c]);
    }
  } else if (MODE == OUT_ADERB) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const long long idx = base + c * NODES;
      args.out[idx] = args.v[idx] - res[c];
    }
  }
}

}  // namespace wk
