// FP64 peak microbenchmark: DFMA pipe throughput and DMMA (mma.sync m8n8k4 f64).
// Writes one JSON line per measurement.  Used to set the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - a;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
    }
  }
  double s = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 256;
    dfma_loop<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("{\"kind\": \"dfma\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", bpsm, ms, flops / ms / 1e9);
  }
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 256;
    dmma_loop<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 32.0 * iters * (double)blocks * threads / 32;
    printf("{\"kind\": \"dmma\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", bpsm, ms, flops / ms / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 4 GiB per buffer in double2
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 256>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kind\": \"copy\", \"GBps\": %.1f}\n", 2.0 * n * 16 / ms / 1e6);
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
