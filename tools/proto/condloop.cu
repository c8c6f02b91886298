// Per-iteration overhead of a cudaGraphCondTypeWhile loop and of a last-block
// grid reduction (nvcc -O3 -gencode arch=compute_100a,code=sm_100a condloop.cu).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_step(int* it, int n, cudaGraphConditionalHandle h) {
  const int v = ++*it;
  cudaGraphSetConditional(h, v < n ? 1u : 0u);
}
__global__ void k_noop(double* x) { if (threadIdx.x == 1000) x[0] = 1; }
__global__ void k_red(const double* __restrict__ a, long long n, double* part, unsigned* cnt, double* res) {
  __shared__ double ws[32];
  __shared__ bool last;
  double v = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) v += a[i] * a[i];
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < blockDim.x / 32 ? ws[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(~0u, v, o);
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double s = 0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += ((volatile double*)part)[i];
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(~0u, s, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) { double t = 0; for (int w = 0; w < blockDim.x / 32; ++w) t += ws[w]; *res = t; *cnt = 0; }
  }
}
// last-block pattern with one acq_rel atomic (no separate __threadfence round trip)
__global__ void k_red3(const double* __restrict__ a, long long n, double* part, unsigned* cnt, double* res) {
  __shared__ double ws[32];
  __shared__ bool last;
  double v = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) v += a[i] * a[i];
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < blockDim.x / 32 ? ws[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(~0u, v, o);
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = v;
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    last = old == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    double s = 0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += ((volatile double*)part)[i];
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(~0u, s, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) { double t = 0; for (int w = 0; w < blockDim.x / 32; ++w) t += ws[w]; *res = t; *cnt = 0; }
  }
}
// block partials written, no last-block pass (a second 1-block kernel sums them)
__global__ void k_red2(const double* __restrict__ a, long long n, double* part) {
  __shared__ double ws[32];
  double v = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) v += a[i] * a[i];
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) { double t = 0; for (int w = 0; w < blockDim.x / 32; ++w) t += ws[w]; part[blockIdx.x] = t; }
}
__global__ void k_sq(const double* __restrict__ a, long long n, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) out[i] = a[i] * a[i];
}

int main() {
  cudaStream_t s, s2;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  int* it; double* x; CK(cudaMalloc(&it, 4)); CK(cudaMalloc(&x, 16 << 20));
  const long long n = 616962;
  double *part, *res; unsigned* cnt;
  CK(cudaMalloc(&part, 4096 * 8)); CK(cudaMalloc(&res, 8)); CK(cudaMalloc(&cnt, 4)); CK(cudaMemset(cnt, 0, 4));
  CK(cudaMemset(x, 0, 16 << 20));
  for (int nk = 0; nk <= 8; nk += 4) {
    for (int variant = 0; variant < 7; ++variant) {
      const int N = 2000;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
      cudaStreamCaptureStatus st; cudaGraph_t g; const cudaGraphNode_t* deps; size_t nd;
      CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
      cudaGraphConditionalHandle h;
      CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
      CK(cudaMemsetAsync(it, 0, 4, s));
      CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
      cudaGraphNode_t cn;
      CK(cudaGraphAddNode(&cn, g, deps, nd, &cp));
      CK(cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies));
      CK(cudaStreamBeginCaptureToGraph(s2, cp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeGlobal));
      for (int k = 0; k < nk; ++k) {
        if (variant == 0) k_noop<<<1, 32, 0, s2>>>(x);
        else if (variant == 1) k_red<<<1184, 256, 0, s2>>>(x, n, part, cnt, res);
        else if (variant == 2) k_sq<<<1184, 256, 0, s2>>>(x, n, x + n);
        else if (variant == 3) k_red<<<296, 256, 0, s2>>>(x, n, part, cnt, res);
        else if (variant == 4) k_red2<<<296, 256, 0, s2>>>(x, n, part);
        else if (variant == 5) k_red3<<<296, 256, 0, s2>>>(x, n, part, cnt, res);
        else k_red3<<<1184, 256, 0, s2>>>(x, n, part, cnt, res);
      }
      k_step<<<1, 1, 0, s2>>>(it, N, h);
      cudaGraph_t bo; CK(cudaStreamEndCapture(s2, &bo));
      cudaGraph_t go; CK(cudaStreamEndCapture(s, &go));
      cudaGraphExec_t ge; CK(cudaGraphInstantiate(&ge, go, 0));
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      CK(cudaGraphLaunch(ge, s));
      cudaEventRecord(a, s); CK(cudaGraphLaunch(ge, s)); cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      const char* nm[7] = {"noop 1-block", "reduce 1184 blk (last-block)", "square 616962 (no reduce)",
                           "reduce 296 blk (last-block)", "reduce 296 blk (partials only)",
                           "reduce 296 blk (acq_rel atom)", "reduce 1184 blk (acq_rel atom)"};
      printf("while loop, %d x %-28s + step kernel: %.2f us/iter\n", nk, nm[variant], 1e3 * ms / N);
      if (nk == 0) break;
    }
  }
  return 0;
}
