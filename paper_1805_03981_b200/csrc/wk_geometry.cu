// Curved-cell geometry on the device: the GeometryCache arrays
// (reference mesh.py:245-334, precompute_geometry / _volume_geometry /
// _face_geometry) evaluated from the nodal coordinates of the geometry map.
//
// For a tensor point set (p_0, .., p_{d-1}) of per-direction Lagrange rows
// val_m, der_m of the degree-g GL basis, one thread per point computes
//   J[i][m] = d x_i / d xi_m = sum_nodes X_i(node) prod_j (j == m ? der_j : val_j)
// directly from the element's nodes (staged in shared memory; one CTA per
// element), its determinant and inverse, and writes
//   volume:   inv_jac[e][m][i][pt] = (J^{-1})[m][i],  jxw[e][pt] = det * w(pt)
//   face m,s: n = (2s-1) det J^{-T} e_m,  normal[e][i][pt] = n_i / |n|,
//             jxw[e][pt] = |n| * w(pt)
// (the reference's formulas, mesh.py:249-286).  The volume pass also reports
// per element max|J - J(first point)|, max|offdiagonal J|, max|J| for the
// reference's cartesian_flag, and flags det <= 0 (the reference raises).
// Setup-only: ~(g+1)^d * 13 flops per point.
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
  const double* nodes;            // (E, d, (g+1)^d), direction 0 fastest
  double* inv_jac;                // volume: (E, d, d, P)
  double* jxw;                    // (E, P)
  double* normal;                 // face: (E, d, P)
  double* stats;                  // volume: (E, 3) or null
  int* bad;                       // det <= 0 flag or null
  long long E;
  int g1;                         // g + 1
  int np[3];                      // points per direction
  int face_axis, face_side;       // face_axis < 0: volume
  const double* tab;              // device: val[3][kT] | der[3][kT] | w[kW]
};
constexpr int kT = kPMax * kGMax;               // [m][p * g1 + a]
constexpr int kW = kPMax * kPMax * kPMax;
constexpr int kTab = 6 * kT + kW;

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* slot, double v) {
  atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

template <int D>
__global__ void metric_kernel(const __grid_constant__ MetricArgs A) {
  extern __shared__ double xs[];              // (D, g1^D) | J at point 0 | 3 stats
  const long long e = blockIdx.x;
  const int g1 = A.g1;
  const int nn = D == 3 ? g1 * g1 * g1 : g1 * g1;
  const int P = D == 3 ? A.np[0] * A.np[1] * A.np[2] : A.np[0] * A.np[1];
  double* tb = xs + D * nn;                   // the point tables (from global)
  double* J0 = tb + kTab;
  unsigned long long* st = reinterpret_cast<unsigned long long*>(J0 + D * D);
  for (int t = threadIdx.x; t < kTab; t += blockDim.x) tb[t] = A.tab[t];
  const double* val = tb;
  const double* der = tb + 3 * kT;
  const double* wq = tb + 6 * kT;
  for (int t = threadIdx.x; t < D * nn; t += blockDim.x) xs[t] = A.nodes[e * D * nn + t];
  if (threadIdx.x < 3) st[threadIdx.x] = 0ull;
  __syncthreads();
  const int pt = threadIdx.x;
  double J[D][D] = {};
  const bool live = pt < P;
  if (!live) {            // idle lanes: identity (keeps the inverse finite)
#pragma unroll
    for (int i = 0; i < D; ++i) J[i][i] = 1.0;
  } else {
    const int p0 = pt % A.np[0];
    const int p1 = (pt / A.np[0]) % A.np[1];
    const int p2 = D == 3 ? pt / (A.np[0] * A.np[1]) : 0;
    const int nc = D == 3 ? g1 : 1;
    for (int c = 0; c < nc; ++c) {
      const double v2 = D == 3 ? val[2 * kT + p2 * g1 + c] : 1.0;
      const double d2 = D == 3 ? der[2 * kT + p2 * g1 + c] : 0.0;
      for (int b = 0; b < g1; ++b) {
        const double v1 = val[kT + p1 * g1 + b], d1 = der[kT + p1 * g1 + b];
        const double tvv = v1 * v2, tdv = d1 * v2, tvd = v1 * d2;
        const int base = (c * g1 + b) * g1;
        for (int a = 0; a < g1; ++a) {
          const double v0 = val[p0 * g1 + a], d0 = der[p0 * g1 + a];
          const double w0 = d0 * tvv, w1 = v0 * tdv, w2 = v0 * tvd;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const double x = xs[i * nn + base + a];
            J[i][0] = fma(w0, x, J[i][0]);
            J[i][1] = fma(w1, x, J[i][1]);
            if (D == 3) J[i][D - 1] = fma(w2, x, J[i][D - 1]);
          }
        }
      }
    }
  }
  double det, inv[D][D];
  if (D == 3) {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    const double r = 1.0 / det;
    // (J^{-1})[m][i] = cof(J)[i][m] / det
    inv[0][0] = c00 * r;
    inv[1][0] = c01 * r;
    inv[2][0] = c02 * r;
    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * r;
    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * r;
    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * r;
    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * r;
    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * r;
    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * r;
  } else {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double r = 1.0 / det;
    inv[0][0] = J[1][1] * r;
    inv[0][1] = -J[0][1] * r;
    inv[1][0] = -J[1][0] * r;
    inv[1][1] = J[0][0] * r;
  }
  if (live && !(det > 0.0) && A.bad) atomicExch(A.bad, 1);
  if (A.face_axis < 0) {
    if (live) {
#pragma unroll
      for (int m = 0; m < D; ++m)
#pragma unroll
        for (int i = 0; i < D; ++i) A.inv_jac[((e * D + m) * D + i) * P + pt] = inv[m][i];
      A.jxw[e * P + pt] = det * wq[pt];
    }
    if (A.stats) {
      if (pt == 0) {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int m = 0; m < D; ++m) J0[i * D + m] = J[i][m];
      }
      __syncthreads();
      if (live) {
        double dev = 0.0, off = 0.0, mx = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int m = 0; m < D; ++m) {
            dev = fmax(dev, fabs(J[i][m] - J0[i * D + m]));
            if (i != m) off = fmax(off, fabs(J[i][m]));
            mx = fmax(mx, fabs(J[i][m]));
          }
        atomic_max_nonneg(&st[0], dev);
        atomic_max_nonneg(&st[1], off);
        atomic_max_nonneg(&st[2], mx);
      }
      __syncthreads();
      if (threadIdx.x < 3) A.stats[e * 3 + threadIdx.x] = __longlong_as_double((long long)st[threadIdx.x]);
    }
  } else if (live) {
    const int m = A.face_axis;
    const double sgn = 2.0 * A.face_side - 1.0;
    double nv[D], len2 = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      // row m of J^{-1}, selected with compile-time indices (no local memory)
      double r = inv[0][i];
#pragma unroll
      for (int mm = 1; mm < D; ++mm) r = (m == mm) ? inv[mm][i] : r;
      nv[i] = sgn * det * r;
      len2 = fma(nv[i], nv[i], len2);
    }
    const double len = sqrt(len2);
#pragma unroll
    for (int i = 0; i < D; ++i) A.normal[(e * D + i) * P + pt] = nv[i] / len;
    A.jxw[e * P + pt] = len * wq[pt];
  }
}

}  // namespace
}  // namespace wk

using namespace wk;

extern "C" int wk_curved_metric(int d, int g, int64_t E, const double* nodes,
                                const int32_t* npts, const double* val, const double* der,
                                const double* wts, int face_axis, int face_side, double* inv_jac,
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
      std::memcpy(&tab[m * kT], val + off, sizeof(double) * npts[m] * (g + 1));
      std::memcpy(&tab[(3 + m) * kT], der + off, sizeof(double) * npts[m] * (g + 1));
      off += npts[m] * (g + 1);
    }
    if (d == 2) a.np[2] = 1;
    std::memcpy(&tab[6 * kT], wts, sizeof(double) * P);
    require(face_axis >= 0 ? (normal && jxw) : (inv_jac && jxw), "missing output array");
    if (E == 0) return;
    const int threads = ((P + 31) / 32) * 32;
    const int nn = d == 3 ? (g + 1) * (g + 1) * (g + 1) : (g + 1) * (g + 1);
    const size_t smem = sizeof(double) * (d * nn + kTab + d * d + 3);
    auto s = (cudaStream_t)stream;
    // the point tables travel through a small device buffer (setup-only)
    double* dtab = nullptr;
    WK_CUDA(cudaMalloc(&dtab, sizeof(double) * kTab));
    WK_CUDA(cudaMemcpyAsync(dtab, tab.data(), sizeof(double) * kTab, cudaMemcpyHostToDevice, s));
    a.tab = dtab;
    if (d == 3) metric_kernel<3><<<(unsigned)E, threads, smem, s>>>(a);
    else metric_kernel<2><<<(unsigned)E, threads, smem, s>>>(a);
    WK_CUDA_AT(cudaGetLastError(), "metric_kernel");
    WK_CUDA(cudaStreamSynchronize(s));
    WK_CUDA(cudaFree(dtab));
  });
}
