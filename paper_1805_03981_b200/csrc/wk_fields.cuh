// Field-level kernels around the time loop: the
// mass-weighted state norm (stepping.py:321-324), the standing-mode initial
// state (analytic.py:48-64) and the L2 pressure error (analytic.py:67-93).
// None is on the timed path; all are deterministic (per-element partial sums
// reduced in a fixed order by one block, no floating-point atomics).
#pragma once
#include <cuda_runtime.h>

namespace wk {
namespace fields {

constexpr int kMaxQ = 12;            // points per direction (k + 1 + n_extra)
constexpr int kThreads = 128;

// out = M along direction m of a tensor with `ncomp` leading blocks of
// extents ext[0..D) (direction 0 fastest); M is nt x nf (row-major)
template <int D>
static __device__ void sweep(const double* in, double* out, const double* M, int nf, int nt, int m,
                      const int* ext, int ncomp) {
  int ein[3] = {ext[0], ext[1], D == 3 ? ext[2] : 1};
  int eout[3] = {ein[0], ein[1], ein[2]};
  eout[m] = nt;
  const int vin = ein[0] * ein[1] * ein[2], vout = eout[0] * eout[1] * eout[2];
  const int sm = m == 0 ? 1 : (m == 1 ? eout[0] : eout[0] * eout[1]);   // stride in out
  const int sim = m == 0 ? 1 : (m == 1 ? ein[0] : ein[0] * ein[1]);     // stride in in
  for (int t = threadIdx.x; t < ncomp * vout; t += blockDim.x) {
    const int c = t / vout, r = t - c * vout;
    const int i = (r / sm) % nt;
    const int rest = r - i * sm;                 // position with i_m = 0 (out strides)
    // same position in the input: the strides below m agree, above m scale
    const int lo = rest % sm, hi = rest / (sm * nt);
    const double* src = in + c * vin + lo + hi * sim * nf;
    double s = 0.0;
    for (int j = 0; j < nf; ++j) s = fma(M[i * nf + j], src[j * sim], s);
    out[t] = s;
  }
}

// sum of block values -> thread 0 (shared scratch of blockDim doubles)
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  scratch[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) scratch[threadIdx.x] += scratch[threadIdx.x + s];
    __syncthreads();
  }
  const double r = scratch[0];
  __syncthreads();
  return r;
}

// out[0] = sum(part[0..n)) in a fixed order (one block)
static __global__ void ordered_sum_kernel(const double* part, long long n, double* out) {
  __shared__ double scratch[kThreads];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) out[0] = s;
}

// per element: sum_{c, q} JxW_q (B^{(x)D} u_c)_q^2.  JxW: per point array
// (curved) or det[class] * prod w (affine).
template <int D>
__global__ void mass_norm_kernel(const double* u, int n, const double* Bg, const double* w,
                                 const double* jxw, const double* geo, int geo_stride,
                                 int det_off, const int* cls, double* part) {
  extern __shared__ double sm[];
  const long long e = blockIdx.x;
  const int C = D + 1, nodes = D == 3 ? n * n * n : n * n;
  double* a = sm;
  double* b = a + C * nodes;
  double* B = b + C * nodes;
  double* scratch = B + n * n;
  for (int t = threadIdx.x; t < C * nodes; t += blockDim.x) a[t] = u[e * C * nodes + t];
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) B[t] = Bg[t];
  __syncthreads();
  int ext[3] = {n, n, n};
  double* cur = a;
  double* nxt = b;
  for (int m = 0; m < D; ++m) {
    sweep<D>(cur, nxt, B, n, n, m, ext, C);
    __syncthreads();
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  const double det = jxw ? 0.0 : geo[(cls ? cls[e] : 0) * geo_stride + det_off];
  double s = 0.0;
  for (int t = threadIdx.x; t < C * nodes; t += blockDim.x) {
    const int q = t % nodes;
    double wq;
    if (jxw) {
      wq = jxw[e * nodes + q];
    } else {
      const int q0 = q % n, q1 = (q / n) % n;
      wq = det * w[q0] * w[q1];
      if (D == 3) wq *= w[q / (n * n)];
    }
    s = fma(wq * cur[t], cur[t], s);
  }
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) part[e] = s;
}

}  // namespace fields
}  // namespace wk
