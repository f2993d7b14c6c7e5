// Runtime-sized element-local kernels behind the reference's non-fused
// operator API (operator.py:250-325): mass / inverse mass, GL<->Gauss basis
// changes, degree resize, pointwise local S.  One block per element, the
// element's (C, n^d) tile staged in shared memory.  These serve the drop-in
// API and the composed (unfused) stepping path; the timed hot path uses the
// fused kernels in wk_affine.cuh / wk_tck.cuh / wk_curved.cuh.
#pragma once
#include "wk_common.cuh"

namespace wk {

enum ScaleMode : int {
  SCALE_NONE = 0,
  SCALE_DET = 1,       // x * det J        (affine class record)
  SCALE_INV_DET = 2,   // x / det J
  SCALE_MUL_PTS = 3,   // x * w[e, pt]     (per-point array, e.g. JxW)
  SCALE_DIV_PTS = 4,   // x / w[e, pt]
};

struct SweepArgs {
  const double* in;
  double* out;
  const double* mat;     // (nt, nf) row-major, same in every direction
  const double* pts;     // per-point scale array (E, npts) for *_PTS modes
  const double* geo;     // affine class records (for det)
  const int* geo_class;
  int geo_stride, det_off;
  long long E;
  int D, C, nf, nt;
  int pre_mode;          // applied to the input (at nf points)
  int post_mode;         // applied to the output (at nt points)
  double out_scale;      // final multiplier (e.g. -1)
};

__device__ __forceinline__ double elem_det(const SweepArgs& a, long long e) {
  const int cls = a.geo_class ? __ldg(a.geo_class + e) : 0;
  return __ldg(a.geo + (long long)cls * a.geo_stride + a.det_off);
}

__global__ void sweep_all_kernel(SweepArgs a) {
  extern __shared__ double sm[];
  const long long e = blockIdx.x;
  const int D = a.D, C = a.C, nf = a.nf, nt = a.nt;
  const int nmax = nf > nt ? nf : nt;
  const int cap = D == 3 ? nmax * nmax * nmax : nmax * nmax;
  double* buf0 = sm;
  double* buf1 = sm + C * cap;
  double* mat = buf1 + C * cap;
  for (int i = threadIdx.x; i < nt * nf; i += blockDim.x) mat[i] = a.mat[i];
  const int nin = D == 3 ? nf * nf * nf : nf * nf;
  const int nout = D == 3 ? nt * nt * nt : nt * nt;
  double det = 1.0;
  if (a.pre_mode == SCALE_DET || a.pre_mode == SCALE_INV_DET || a.post_mode == SCALE_DET ||
      a.post_mode == SCALE_INV_DET)
    det = elem_det(a, e);
  for (int t = threadIdx.x; t < C * nin; t += blockDim.x) {
    const int c = t / nin, pt = t - c * nin;
    double x = a.in[(e * C + c) * nin + pt];
    if (a.pre_mode == SCALE_DET) x *= det;
    else if (a.pre_mode == SCALE_INV_DET) x /= det;
    else if (a.pre_mode == SCALE_MUL_PTS) x *= a.pts[e * nin + pt];
    else if (a.pre_mode == SCALE_DIV_PTS) x /= a.pts[e * nin + pt];
    buf0[c * cap + pt] = x;
  }
  __syncthreads();
  double* cur = buf0;
  double* nxt = buf1;
  for (int m = 0; m < D; ++m) {
    int ein[3] = {1, 1, 1}, eout[3] = {1, 1, 1};
    for (int q = 0; q < D; ++q) {
      ein[q] = q < m ? nt : nf;
      eout[q] = q <= m ? nt : nf;
    }
    const int tot = eout[0] * eout[1] * eout[2];
    const int sin_m = m == 0 ? 1 : (m == 1 ? ein[0] : ein[0] * ein[1]);
    for (int t = threadIdx.x; t < C * tot; t += blockDim.x) {
      const int c = t / tot, pt = t - c * tot;
      const int idx[3] = {pt % eout[0], (pt / eout[0]) % eout[1], pt / (eout[0] * eout[1])};
      int lin = 0, stride = 1;
      for (int q = 0; q < D; ++q) {
        if (q != m) lin += idx[q] * stride;
        stride *= ein[q];
      }
      const double* src = cur + c * cap + lin;
      const double* row = mat + idx[m] * nf;
      double s = 0.0;
      for (int j = 0; j < nf; ++j) s = fma(row[j], src[j * sin_m], s);
      nxt[c * cap + pt] = s;
    }
    __syncthreads();
    double* tt = cur; cur = nxt; nxt = tt;
  }
  for (int t = threadIdx.x; t < C * nout; t += blockDim.x) {
    const int c = t / nout, pt = t - c * nout;
    double x = cur[c * cap + pt];
    if (a.post_mode == SCALE_DET) x *= det;
    else if (a.post_mode == SCALE_INV_DET) x /= det;
    else if (a.post_mode == SCALE_MUL_PTS) x *= a.pts[e * nout + pt];
    else if (a.post_mode == SCALE_DIV_PTS) x /= a.pts[e * nout + pt];
    a.out[(e * C + c) * nout + pt] = a.out_scale * x;
  }
}

struct LocalSArgs {
  const double* in;      // (E, C, nq^D) collocated Gauss values
  double* out;
  const double* dco;     // (nq, nq) collocation derivative
  const double* geo;     // affine class records (G at offset 0) or null
  const int* geo_class;
  int geo_stride;
  const double* inv_jac; // curved: (E, D, D, nq^D) or null
  const double* mat;     // (E, kMatStride)
  long long E;
  int D, nq;
};

// apply_local_S (operator.py:286-306): pointwise S at one degree's Gauss points.
__global__ void local_S_kernel(LocalSArgs a) {
  extern __shared__ double sm[];
  const long long e = blockIdx.x;
  const int D = a.D, C = D + 1, nq = a.nq;
  const int np = D == 3 ? nq * nq * nq : nq * nq;
  double* v = sm;
  double* dm = v + C * np;
  for (int i = threadIdx.x; i < nq * nq; i += blockDim.x) dm[i] = a.dco[i];
  for (int t = threadIdx.x; t < C * np; t += blockDim.x) v[t] = a.in[e * C * np + t];
  __syncthreads();
  const double ir = a.mat[e * kMatStride + 0], c2r = a.mat[e * kMatStride + 1];
  const double* g = nullptr;
  if (a.geo) g = a.geo + (long long)(a.geo_class ? a.geo_class[e] : 0) * a.geo_stride;
  for (int pt = threadIdx.x; pt < np; pt += blockDim.x) {
    double grad[3][4];
    int sm_ = 1;
    for (int m = 0; m < D; ++m) {
      const int im = (pt / sm_) % nq;
      const int base = pt - im * sm_;
      for (int c = 0; c < C; ++c) {
        double s = 0.0;
        for (int j = 0; j < nq; ++j) s = fma(dm[im * nq + j], v[c * np + base + j * sm_], s);
        grad[m][c] = s;
      }
      sm_ *= nq;
    }
    double res[4] = {0.0, 0.0, 0.0, 0.0};
    for (int m = 0; m < D; ++m)
      for (int i = 0; i < D; ++i) {
        const double gmi = g ? g[m * D + i]
                             : a.inv_jac[((e * D + m) * D + i) * (long long)np + pt];
        res[i] = fma(gmi, grad[m][D], res[i]);
        res[D] = fma(gmi, grad[m][i], res[D]);
      }
    for (int i = 0; i < D; ++i) a.out[(e * C + i) * np + pt] = ir * res[i];
    a.out[(e * C + D) * np + pt] = c2r * res[D];
  }
}

// v = u - s * w over n doubles (ADER-HDG V on the general affine path)
__global__ void axpy_kernel(const double* __restrict__ u, const double* __restrict__ w,
                            double* __restrict__ v, double s, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = u[i] - s * w[i];
}

}  // namespace wk
