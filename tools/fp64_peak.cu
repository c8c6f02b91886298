// Measured FP64 (CUDA-core DFMA) peak of the GPU this runs on -- the roofline
// denominator for FP64-bound kernels (MEASURED_PEAKS.json carries only HBM and
// bf16 figures).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak            -> one JSON line (best of 10 runs, CUDA events)
//
// Every thread runs 8 independent DFMA chains (enough ILP to cover the pipe
// latency at full occupancy); 2 flops per DFMA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dfma<<<blocks, threads>>>(out, 64, 0.999999, 1e-9);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  const double tfs = flops / (best * 1e-3) / 1e12;
  std::printf("{\"fp64_dfma_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"sm_clock_mhz_attr\": %d, "
              "\"how\": \"%d blocks x %d threads x 8 independent DFMA chains x %d x 16, best of 10, CUDA events\"}\n",
              tfs, best, sms, clk / 1000, blocks, threads, iters);
  cudaError_t err = cudaGetLastError();
  return err == cudaSuccess ? 0 : 1;
}
