// Curved-cell geometry on the device: the GeometryCache arrays
// (reference mesh.py:245-334, precompute_geometry / _volume_geometry /
// _face_geometry) evaluated from the nodal coordinates of the geometry map.
//
// For a tensor point set (p_0, .., p_{d-1}) of per-direction Lagrange rows
// val_m, der_m of the degree-g GL basis, one thread per point computes
//   J[i][m] = d x_i / d xi_m = sum_nodes X_i(node) prod_j (j == m ? der_j : val_j)
// directly from the element's nodes (staged in shared memory; one CTA per
// element), its adjugate, determinant and inverse, and writes
//   volume:   inv_jac[e][m][i][pt] = (J^{-1})[m][i],  jxw[e][pt] = det * w(pt)
//   face m,s: n = (2s-1) det J^{-T} e_m,  normal[e][i][pt] = n_i / |n|,
//             jxw[e][pt] = |n| * w(pt)
// (the reference's formulas, mesh.py:249-286).  The volume pass also reports
// per element max|J - J(first point)|, max|offdiagonal J|, max|J| for the
// reference's cartesian_flag, and flags det <= 0 (the reference raises).
//
// The nodal coordinates arrive as double-double pairs too (hi array, then lo
// array): the host evaluates the map in long double and does not round it.
//
// Precision: J ~ h (1/32 at config 3) is a sum of coordinates ~1 times
// derivative rows ~20 whose exact sum is zero.  In plain double the rounding
// of the rows and the summation order leave ~|x|/h * 1e-16 ~ 1e-13 relative
// error, which is implementation-dependent and, near config 3's pulse, moves
// rhs by ~1e-11.  So everything is evaluated in DOUBLE-DOUBLE from rows given
// as hi + lo pairs (long double on the host) and rounded once: the result is
// the correctly rounded metric of the interpolated map to ~1 ulp, the same
// value the host builder computes in long double (mesh.py _metric) and the
// oracle (oracle/mesh.py).  Setup-only (~30 dd flops per node and point).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/wavekernel_b200.h"
#include "wk_error.h"

namespace wk {
namespace {

constexpr int kGMax = 9;          // g + 1 <= 9
constexpr int kPMax = 9;          // points per direction <= 9

struct MetricArgs {
  const double* nodes;            // hi (E, d, (g+1)^d), direction 0 fastest, then lo (same)
  double* inv_jac;                // volume: (E, d, d, P)
  double* jxw;                    // (E, P)
  double* normal;                 // face: (E, d, P)
  double* stats;                  // volume: (E, 3) or null
  int* bad;                       // det <= 0 flag or null
  long long E;
  int g1;                         // g + 1
  int np[3];                      // points per direction
  int face_axis, face_side;       // face_axis < 0: volume
  const double* tab;              // device: val hi|lo [3][kT], der hi|lo [3][kT], w[kW]
};
constexpr int kT = kPMax * kGMax;               // [m][p * g1 + a]
constexpr int kW = kPMax * kPMax * kPMax;
constexpr int kTab = 12 * kT + kW;

// ---- double-double arithmetic (hi + lo, |lo| <= ulp(hi) / 2) --------------
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd fast_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ dd add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  const dd t = two_sum(x.lo, y.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd mul(dd x, dd y) {
  const double p = __dmul_rn(x.hi, y.hi);
  double e = __fma_rn(x.hi, y.hi, -p);
  e = __fma_rn(x.hi, y.lo, e);
  e = __fma_rn(x.lo, y.hi, e);
  return fast_two_sum(p, e);
}
__device__ __forceinline__ dd mul(dd x, double y) {
  const double p = __dmul_rn(x.hi, y);
  const double e = __fma_rn(x.lo, y, __fma_rn(x.hi, y, -p));
  return fast_two_sum(p, e);
}
__device__ __forceinline__ dd div(dd x, dd y) {
  const double q1 = __ddiv_rn(x.hi, y.hi);
  const dd r = add(x, neg(mul(y, q1)));
  const double q2 = __ddiv_rn(r.hi, y.hi);
  const dd r2 = add(r, neg(mul(y, q2)));
  const double q3 = __ddiv_rn(r2.hi, y.hi);
  return add(fast_two_sum(q1, q2), dd{q3, 0.0});
}
__device__ __forceinline__ dd sqrt_dd(dd x) {
  const double s = sqrt(x.hi);
  const double p = __dmul_rn(s, s);
  const dd r = add(x, neg(dd{p, __fma_rn(s, s, -p)}));
  return fast_two_sum(s, __ddiv_rn(r.hi, 2.0 * s));
}
__device__ __forceinline__ double rnd(dd x) { return __dadd_rn(x.hi, x.lo); }

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* slot, double v) {
  atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

template <int D>
__global__ void metric_kernel(const __grid_constant__ MetricArgs A) {
  extern __shared__ double xs[];              // hi (D, g1^D) | lo | tables | J at point 0 | stats
  const long long e = blockIdx.x;
  const int g1 = A.g1;
  const int nn = D == 3 ? g1 * g1 * g1 : g1 * g1;
  const int P = D == 3 ? A.np[0] * A.np[1] * A.np[2] : A.np[0] * A.np[1];
  double* tb = xs + 2 * D * nn;               // the point tables (from global)
  double* J0 = tb + kTab;
  unsigned long long* st = reinterpret_cast<unsigned long long*>(J0 + D * D);
  for (int t = threadIdx.x; t < kTab; t += blockDim.x) tb[t] = A.tab[t];
  const double* vhi = tb;
  const double* vlo = tb + 3 * kT;
  const double* dhi = tb + 6 * kT;
  const double* dlo = tb + 9 * kT;
  const double* wq = tb + 12 * kT;
  for (int t = threadIdx.x; t < D * nn; t += blockDim.x) {
    xs[t] = A.nodes[e * D * nn + t];
    xs[D * nn + t] = A.nodes[(A.E + e) * D * nn + t];
  }
  if (threadIdx.x < 3) st[threadIdx.x] = 0ull;
  __syncthreads();
  // the points of the element in passes of blockDim.x (uniform trip count:
  // the barrier inside the stats pass is reached by every thread)
  for (int pt0 = 0; pt0 < P; pt0 += blockDim.x) {
    const int pt = pt0 + threadIdx.x;
    dd J[D][D];
    #pragma unroll
    for (int i = 0; i < D; ++i)
      #pragma unroll
      for (int m = 0; m < D; ++m) J[i][m] = {i == m ? 1.0 : 0.0, 0.0};
    const bool live = pt < P;
    if (live) {
      #pragma unroll
      for (int i = 0; i < D; ++i) J[i][i] = {0.0, 0.0};
      const int p0 = pt % A.np[0];
      const int p1 = (pt / A.np[0]) % A.np[1];
      const int p2 = D == 3 ? pt / (A.np[0] * A.np[1]) : 0;
      const int nc = D == 3 ? g1 : 1;
      for (int c = 0; c < nc; ++c) {
        const dd v2 = D == 3 ? dd{vhi[2 * kT + p2 * g1 + c], vlo[2 * kT + p2 * g1 + c]} : dd{1.0, 0.0};
        const dd d2 = D == 3 ? dd{dhi[2 * kT + p2 * g1 + c], dlo[2 * kT + p2 * g1 + c]} : dd{0.0, 0.0};
        for (int b = 0; b < g1; ++b) {
          const dd v1 = {vhi[kT + p1 * g1 + b], vlo[kT + p1 * g1 + b]};
          const dd d1 = {dhi[kT + p1 * g1 + b], dlo[kT + p1 * g1 + b]};
          const dd tvv = mul(v1, v2), tdv = mul(d1, v2), tvd = mul(v1, d2);
          const int base = (c * g1 + b) * g1;
          for (int a = 0; a < g1; ++a) {
            const dd v0 = {vhi[p0 * g1 + a], vlo[p0 * g1 + a]};
            const dd d0 = {dhi[p0 * g1 + a], dlo[p0 * g1 + a]};
            const dd w0 = mul(d0, tvv), w1 = mul(v0, tdv), w2 = mul(v0, tvd);
            #pragma unroll
            for (int i = 0; i < D; ++i) {
              const dd x = {xs[i * nn + base + a], xs[(D + i) * nn + base + a]};
              J[i][0] = add(J[i][0], mul(w0, x));
              J[i][1] = add(J[i][1], mul(w1, x));
              if (D == 3) J[i][D - 1] = add(J[i][D - 1], mul(w2, x));
            }
          }
        }
      }
    }
    // cof[i][m] = det J * (J^{-1})[m][i]: column m of cof is det J^{-T} e_m
    dd cof[D][D], det;
    if (D == 3) {
      #pragma unroll
      for (int i = 0; i < 3; ++i)
        #pragma unroll
        for (int m = 0; m < 3; ++m) {
          const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, m1 = (m + 1) % 3, m2 = (m + 2) % 3;
          cof[i][m] = add(mul(J[i1][m1], J[i2][m2]), neg(mul(J[i1][m2], J[i2][m1])));
        }
      det = add(add(mul(J[0][0], cof[0][0]), mul(J[0][1], cof[0][1])), mul(J[0][2], cof[0][2]));
    } else {
      cof[0][0] = J[1][1];
      cof[0][1] = neg(J[1][0]);
      cof[1][0] = neg(J[0][1]);
      cof[1][1] = J[0][0];
      det = add(mul(J[0][0], J[1][1]), neg(mul(J[0][1], J[1][0])));
    }
    const double det_r = rnd(det);
    if (live && !(det_r > 0.0) && A.bad) atomicExch(A.bad, 1);
    if (A.face_axis < 0) {
      if (live) {
        #pragma unroll
        for (int m = 0; m < D; ++m)
          #pragma unroll
          for (int i = 0; i < D; ++i)
            A.inv_jac[((e * D + m) * D + i) * P + pt] = rnd(div(cof[i][m], det));
        A.jxw[e * P + pt] = rnd(mul(det, wq[pt]));
      }
      if (A.stats) {
        if (pt == 0) {   // first pass: point 0's J, read by every later point
          #pragma unroll
          for (int i = 0; i < D; ++i)
            #pragma unroll
            for (int m = 0; m < D; ++m) J0[i * D + m] = rnd(J[i][m]);
        }
        __syncthreads();
        if (live) {
          double dev = 0.0, off = 0.0, mx = 0.0;
          #pragma unroll
          for (int i = 0; i < D; ++i)
            #pragma unroll
            for (int m = 0; m < D; ++m) {
              const double jr = rnd(J[i][m]);
              dev = fmax(dev, fabs(jr - J0[i * D + m]));
              if (i != m) off = fmax(off, fabs(jr));
              mx = fmax(mx, fabs(jr));
            }
          atomic_max_nonneg(&st[0], dev);
          atomic_max_nonneg(&st[1], off);
          atomic_max_nonneg(&st[2], mx);
        }
      }
    } else if (live) {
      const int m = A.face_axis;
      const double sgn = 2.0 * A.face_side - 1.0;
      dd nv[D], len2 = {0.0, 0.0};
      #pragma unroll
      for (int i = 0; i < D; ++i) {
        // column m of cof, selected with compile-time indices (no local memory)
        dd r = cof[i][0];
        #pragma unroll
        for (int mm = 1; mm < D; ++mm) r = (m == mm) ? cof[i][mm] : r;
        nv[i] = mul(r, sgn);
        len2 = add(len2, mul(nv[i], nv[i]));
      }
      const dd len = sqrt_dd(len2);
      #pragma unroll
      for (int i = 0; i < D; ++i) A.normal[(e * D + i) * P + pt] = rnd(div(nv[i], len));
      A.jxw[e * P + pt] = rnd(mul(len, wq[pt]));
    }
  }
  if (A.face_axis < 0 && A.stats) {
    __syncthreads();
    if (threadIdx.x < 3) A.stats[e * 3 + threadIdx.x] = __longlong_as_double((long long)st[threadIdx.x]);
  }
}

}  // namespace
}  // namespace wk

using namespace wk;

extern "C" int wk_curved_metric(int d, int g, int64_t E, const double* nodes,
                                const int32_t* npts, const double* val_hi, const double* val_lo,
                                const double* der_hi, const double* der_lo, const double* wts, int face_axis, int face_side, double* inv_jac,
                                double* jxw, double* normal, double* stats, int32_t* bad,
                                void* stream) {
  return guarded([&] {
    require(d == 2 || d == 3, "dimension must be 2 or 3");
    require(g >= 1 && g + 1 <= kGMax, "geometry degree out of range (1..8)");
    require(face_axis < d, "bad face axis");
    MetricArgs a;
    std::memset(&a, 0, sizeof(a));
    a.nodes = nodes;
    a.inv_jac = inv_jac;
    a.jxw = jxw;
    a.normal = normal;
    a.stats = stats;
    a.bad = bad;
    a.E = E;
    a.g1 = g + 1;
    a.face_axis = face_axis;
    a.face_side = face_side;
    std::vector<double> tab(kTab, 0.0);
    int P = 1, off = 0;
    for (int m = 0; m < d; ++m) {
      require(npts[m] >= 1 && npts[m] <= kPMax, "points per direction out of range (1..9)");
      a.np[m] = npts[m];
      P *= npts[m];
      const size_t bytes = sizeof(double) * npts[m] * (g + 1);
      std::memcpy(&tab[m * kT], val_hi + off, bytes);
      std::memcpy(&tab[(3 + m) * kT], val_lo + off, bytes);
      std::memcpy(&tab[(6 + m) * kT], der_hi + off, bytes);
      std::memcpy(&tab[(9 + m) * kT], der_lo + off, bytes);
      off += npts[m] * (g + 1);
    }
    if (d == 2) a.np[2] = 1;
    std::memcpy(&tab[12 * kT], wts, sizeof(double) * P);
    require(face_axis >= 0 ? (normal && jxw) : (inv_jac && jxw), "missing output array");
    if (E == 0) return;
    const int threads = P < 256 ? ((P + 31) / 32) * 32 : 256;
    const int nn = d == 3 ? (g + 1) * (g + 1) * (g + 1) : (g + 1) * (g + 1);
    const size_t smem = sizeof(double) * (2 * d * nn + kTab + d * d + 3);
    auto s = (cudaStream_t)stream;
    // the point tables travel through a small device buffer (setup-only)
    double* dtab = nullptr;
    WK_CUDA(cudaMalloc(&dtab, sizeof(double) * kTab));
    WK_CUDA(cudaMemcpyAsync(dtab, tab.data(), sizeof(double) * kTab, cudaMemcpyHostToDevice, s));
    a.tab = dtab;
    if (d == 3) {
      ensure_smem(metric_kernel<3>, smem);
      metric_kernel<3><<<(unsigned)E, threads, smem, s>>>(a);
    } else {
      ensure_smem(metric_kernel<2>, smem);
      metric_kernel<2><<<(unsigned)E, threads, smem, s>>>(a);
    }
    WK_CUDA_AT(cudaGetLastError(), "metric_kernel");
    WK_CUDA(cudaStreamSynchronize(s));
    WK_CUDA(cudaFree(dtab));
  });
}
