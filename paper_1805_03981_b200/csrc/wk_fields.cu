// Standing-mode initial state and L2 pressure error on the device
// (reference analytic.py:24-93).  Element geometry is
// the multilinear vertex map of the mesh (mesh.map_points / _jacobians);
// vertices (E, 2^d, d) with vertex v = sum_j a_j 2^j at corner (a_0, .., a_{d-1}).
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "../../include/wavekernel_b200.h"
#include "wk_basis.h"
#include "wk_error.h"
#include "wk_fields.cuh"

namespace wk {
namespace {

using fields::kMaxQ;
using fields::kThreads;

struct ModeArgs {
  double omega, kx, pamp, vamp;   // w t folded: cos(w t), -(m pi)/(rho w) sin(w t)
};

// multilinear map x(xi) and its Jacobian from the element corners
template <int D>
__device__ __forceinline__ void corner_map(const double* X, const double* xi, double* x,
                                          double (*J)[3]) {
  for (int i = 0; i < D; ++i) {
    x[i] = 0.0;
    if (J)
      for (int m = 0; m < D; ++m) J[i][m] = 0.0;
  }
  for (int v = 0; v < (1 << D); ++v) {
    double N = 1.0, dN[3];
    for (int j = 0; j < D; ++j) {
      const bool a = (v >> j) & 1;
      N *= a ? xi[j] : 1.0 - xi[j];
    }
    if (J) {
      for (int m = 0; m < D; ++m) {
        double p = 1.0;
        for (int j = 0; j < D; ++j) {
          const bool a = (v >> j) & 1;
          p *= (j == m) ? (a ? 1.0 : -1.0) : (a ? xi[j] : 1.0 - xi[j]);
        }
        dN[m] = p;
      }
    }
    for (int i = 0; i < D; ++i) {
      const double c = X[v * D + i];
      x[i] = fma(N, c, x[i]);
      if (J)
        for (int m = 0; m < D; ++m) J[i][m] = fma(dN[m], c, J[i][m]);
    }
  }
}

// analytic.py:24-40: p = cos(w t) prod sin(m pi x_i),
// v_i = -(m pi)/(rho w) sin(w t) cos(m pi x_i) prod_{j != i} sin(m pi x_j)
template <int D>
__device__ __forceinline__ double mode_p(const ModeArgs& M, const double* x) {
  double p = M.pamp;
  for (int i = 0; i < D; ++i) p *= sin(M.kx * x[i]);
  return p;
}

template <int D>
__global__ void mode_state_kernel(long long E, int n, const double* __restrict__ verts,
                                  const double* __restrict__ gl, ModeArgs M, double* out) {
  const int nodes = D == 3 ? n * n * n : n * n;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= E * nodes) return;
  const long long e = t / nodes;
  const int q = (int)(t - e * nodes);
  double xi[3] = {gl[q % n], gl[(q / n) % n], D == 3 ? gl[q / (n * n)] : 0.0};
  double x[3];
  corner_map<D>(verts + e * (1 << D) * D, xi, x, nullptr);
  double s[3], c[3];
  for (int i = 0; i < D; ++i) {
    s[i] = sin(M.kx * x[i]);
    c[i] = cos(M.kx * x[i]);
  }
  double p = M.pamp;
  for (int i = 0; i < D; ++i) p *= s[i];
  double* o = out + e * (D + 1) * nodes + q;
  for (int i = 0; i < D; ++i) {
    double v = M.vamp;
    for (int j = 0; j < D; ++j) v *= (j == i) ? c[j] : s[j];
    o[i * nodes] = v;
  }
  o[D * nodes] = p;
}

// per element: sum_q det J(q) w_q (p_h(q) - p(q))^2 on the nq-point Gauss rule
template <int D>
__global__ void l2_error_kernel(int n, int nq, const double* __restrict__ state,
                                const double* __restrict__ verts, const double* __restrict__ tab,
                                ModeArgs M, double* part) {
  extern __shared__ double sm[];
  const long long e = blockIdx.x;
  const int nodes = D == 3 ? n * n * n : n * n;
  const int qv = D == 3 ? nq * nq * nq : nq * nq;
  double* I = sm;                       // nq x n interpolation GL -> Gauss(nq)
  double* pts = I + nq * n;             // nq points
  double* w = pts + nq;                 // nq weights
  double* a = w + nq;                   // work tiles: max(nodes, qv) each
  const int big = nodes > qv ? nodes : qv;
  double* b = a + big;
  double* scratch = b + big;
  for (int t = threadIdx.x; t < nq * n + 2 * nq; t += blockDim.x) sm[t] = tab[t];
  for (int t = threadIdx.x; t < nodes; t += blockDim.x)
    a[t] = state[(e * (D + 1) + D) * nodes + t];
  __syncthreads();
  int ext[3] = {n, n, n};
  double* cur = a;
  double* nxt = b;
  for (int m = 0; m < D; ++m) {
    fields::sweep<D>(cur, nxt, I, n, nq, m, ext, 1);
    ext[m] = nq;
    __syncthreads();
    double* tt = cur;
    cur = nxt;
    nxt = tt;
  }
  const double* X = verts + e * (1 << D) * D;
  double s = 0.0;
  for (int q = threadIdx.x; q < qv; q += blockDim.x) {
    const int q0 = q % nq, q1 = (q / nq) % nq, q2 = D == 3 ? q / (nq * nq) : 0;
    double xi[3] = {pts[q0], pts[q1], D == 3 ? pts[q2] : 0.0};
    double x[3], J[3][3];
    corner_map<D>(X, xi, x, J);
    double det;
    if (D == 3) {
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
            J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    } else {
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    }
    double wq = w[q0] * w[q1];
    if (D == 3) wq *= w[q2];
    const double d = cur[q] - mode_p<D>(M, x);
    s = fma(det * wq * d, d, s);
  }
  s = fields::block_sum(s, scratch);
  if (threadIdx.x == 0) part[e] = s;
}

ModeArgs mode_args(int d, int m, double t, double c, double rho) {
  ModeArgs M;
  M.omega = c * m * M_PI * std::sqrt((double)d);
  M.kx = m * M_PI;
  M.pamp = std::cos(M.omega * t);
  M.vamp = -(m * M_PI) / (rho * M.omega) * std::sin(M.omega * t);
  return M;
}

}  // namespace
}  // namespace wk

using namespace wk;

extern "C" int wk_mode_state(int d, int k, int64_t E, const double* verts, int m, double t,
                             double c, double rho, double* out, void* stream) {
  return guarded([&] {
    require(d == 2 || d == 3, "dimension must be 2 or 3");
    require(k >= 1 && k <= 8, "degree out of range (1..8)");
    require(m >= 1, "mode must be at least 1");
    if (E == 0) return;
    const int n = k + 1, nodes = d == 3 ? n * n * n : n * n;
    auto s = (cudaStream_t)stream;
    std::vector<double> gl;
    for (long double v : gl_nodes(k)) gl.push_back((double)v);
    double* dgl = nullptr;
    WK_CUDA(cudaMalloc(&dgl, sizeof(double) * n));
    WK_CUDA(cudaMemcpyAsync(dgl, gl.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
    const ModeArgs M = mode_args(d, m, t, c, rho);
    const long long total = E * nodes;
    const unsigned blocks = (unsigned)((total + 255) / 256);
    if (d == 3) mode_state_kernel<3><<<blocks, 256, 0, s>>>(E, n, verts, dgl, M, out);
    else mode_state_kernel<2><<<blocks, 256, 0, s>>>(E, n, verts, dgl, M, out);
    WK_CUDA_AT(cudaGetLastError(), "mode_state_kernel");
    WK_CUDA(cudaStreamSynchronize(s));
    WK_CUDA(cudaFree(dgl));
  });
}

extern "C" int wk_l2_pressure_error(int d, int k, int64_t E, const double* state,
                                    const double* verts, int m, double t, double c, double rho,
                                    int n_extra, double* out_sq, void* stream) {
  return guarded([&] {
    require(d == 2 || d == 3, "dimension must be 2 or 3");
    require(k >= 1 && k <= 8, "degree out of range (1..8)");
    require(n_extra >= 0 && k + 1 + n_extra <= kMaxQ, "error rule too fine");
    auto s = (cudaStream_t)stream;
    if (E == 0) {
      WK_CUDA(cudaMemsetAsync(out_sq, 0, sizeof(double), s));
      return;
    }
    const int n = k + 1, nq = k + 1 + n_extra;
    std::vector<long double> gp, gw;
    gauss_rule(nq, gp, gw);
    Mat I = lagrange(gl_nodes(k), gp, false);   // nq x n
    std::vector<double> tab;
    for (long double v : I) tab.push_back((double)v);
    for (long double v : gp) tab.push_back((double)v);
    for (long double v : gw) tab.push_back((double)v);
    double *dtab = nullptr, *part = nullptr;
    WK_CUDA(cudaMalloc(&dtab, sizeof(double) * tab.size()));
    WK_CUDA(cudaMalloc(&part, sizeof(double) * E));
    WK_CUDA(cudaMemcpyAsync(dtab, tab.data(), sizeof(double) * tab.size(),
                            cudaMemcpyHostToDevice, s));
    const ModeArgs M = mode_args(d, m, t, c, rho);
    const int nodes = d == 3 ? n * n * n : n * n, qv = d == 3 ? nq * nq * nq : nq * nq;
    const int big = nodes > qv ? nodes : qv;
    const size_t smem = sizeof(double) * (nq * n + 2 * nq + 2 * big + kThreads);
    if (d == 3) l2_error_kernel<3><<<(unsigned)E, kThreads, smem, s>>>(n, nq, state, verts, dtab, M, part);
    else l2_error_kernel<2><<<(unsigned)E, kThreads, smem, s>>>(n, nq, state, verts, dtab, M, part);
    WK_CUDA_AT(cudaGetLastError(), "l2_error_kernel");
    fields::ordered_sum_kernel<<<1, kThreads, 0, s>>>(part, E, out_sq);
    WK_CUDA_AT(cudaGetLastError(), "ordered_sum_kernel");
    WK_CUDA(cudaStreamSynchronize(s));
    WK_CUDA(cudaFree(dtab));
    WK_CUDA(cudaFree(part));
  });
}
