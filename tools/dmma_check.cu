// Verifies the m8n8k4 f64 fragment layout assumed by the DMMA sweeps:
//   A (8x4 row):  lane l holds A[l>>2][l&3]
//   B (4x8 col):  lane l holds B[l&3][l>>2]
//   C (8x8):      lane l holds C[l>>2][2*(l&3)+{0,1}]
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* C) {
  int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];
  double b = B[(l & 3) * 8 + (l >> 2)];
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  C[(l >> 2) * 8 + 2 * (l & 3)] = c0;
  C[(l >> 2) * 8 + 2 * (l & 3) + 1] = c1;
}
int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 0.1 * i + 1; hB[i] = 0.3 * i - 2; }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int q = 0; q < 4; ++q) s += hA[i * 4 + q] * hB[q * 8 + j];
      ref[i * 8 + j] = s;
    }
  double *A, *B, *C;
  cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("{\"dmma_layout_maxerr\": %g, \"err\": \"%s\"}\n", err, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
