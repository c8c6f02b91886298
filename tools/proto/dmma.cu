// Check the m8n8k4 f64 mma.sync fragment layout on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* A, const double* B, double* C) {  // A 8x4 row-major, B 4x8 row-major, C 8x8
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];          // A[row=g][k=t]
  double b = B[t * 8 + g];          // B[k=t][col=g]
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  C[g * 8 + 2 * t] = c0;            // C[row=g][col=2t], [2t+1]
  C[g * 8 + 2 * t + 1] = c1;
}
int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i * 0.5 + 1; hB[i] = (i % 7) - 2.5; }
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) { double s = 0; for (int k2 = 0; k2 < 4; ++k2) s += hA[i * 4 + k2] * hB[k2 * 8 + j]; ref[i * 8 + j] = s; }
  double *A, *B, *C; cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, 512, cudaMemcpyDeviceToHost);
  double md = 0; for (int i = 0; i < 64; ++i) md = fmax(md, fabs(hC[i] - ref[i]));
  printf("dmma m8n8k4 max diff %.3e (%s)\n", md, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
