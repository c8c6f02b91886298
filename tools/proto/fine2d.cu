// Prototype timing of level-0 2D Jacobi-sweep variants (matrix-free Q4 K).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fine2d fine2d.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

struct KE { double k[64]; };
constexpr int NX = 961, NY = 321, EXn = 960, EYn = 320;

__host__ __device__ constexpr int corner_of(int dx, int dy) { return dy ? 3 - dx : dx; }
__host__ __device__ constexpr int cx(int m) { return (m == 1 || m == 2) ? 1 : 0; }
__host__ __device__ constexpr int cy(int m) { return m >= 2 ? 1 : 0; }

// ---------------- variant B: direct loads, one node per thread -------------
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_direct(const __grid_constant__ KE ke, const double* __restrict__ x,
    const double* __restrict__ b, const double* __restrict__ dinv, const double* __restrict__ E,
    const uint8_t* __restrict__ mask, double w, double* __restrict__ xo) {
  const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 8 + threadIdx.y;
  if (i >= NX || j >= NY) return;
  double2 xv[9]; unsigned mk[9]; double ev[4];
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const int ii = i + s % 3 - 1, jj = j + s / 3 - 1;
    const bool in = ii >= 0 && ii < NX && jj >= 0 && jj < NY;
    const int n = in ? ii + NX * jj : 0;
    xv[s] = __ldg(reinterpret_cast<const double2*>(x) + n);
    mk[s] = in ? __ldg(mask + n) : 0u;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int ex = i - 1 + (e & 1), ey = j - 1 + (e >> 1);
    const bool in = ex >= 0 && ex < EXn && ey >= 0 && ey < EYn;
    ev[e] = in ? __ldg(E + ex + EXn * ey) : 0.0;
  }
  const int node = i + NX * j;
  const double2 bb = __ldg(reinterpret_cast<const double2*>(b) + node);
  const double2 dd = __ldg(reinterpret_cast<const double2*>(dinv) + node);
  double xs[9][2];
#pragma unroll
  for (int s = 0; s < 9; ++s) { xs[s][0] = (mk[s] & 1) ? xv[s].x : 0.0; xs[s][1] = (mk[s] & 2) ? xv[s].y : 0.0; }
  double acc[2] = {0, 0};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int exo = e & 1, eyo = e >> 1;  // element at (i-1+exo, j-1+eyo)
    const int ln = corner_of(1 - exo, 1 - eyo);
    double t[2] = {0, 0};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int s = (exo + cx(m)) + 3 * (eyo + cy(m));
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int d = 0; d < 2; ++d) t[c] += ke.k[(ln * 2 + c) * 8 + m * 2 + d] * xs[s][d];
    }
    acc[0] += ev[e] * t[0]; acc[1] += ev[e] * t[1];
  }
  const unsigned mn = mk[4];
  const double o0 = (mn & 1) ? acc[0] : xv[4].x, o1 = (mn & 2) ? acc[1] : xv[4].y;
  double2 r;
  r.x = xv[4].x + w * (dd.x * (bb.x - o0));
  r.y = xv[4].y + w * (dd.y * (bb.y - o1));
  reinterpret_cast<double2*>(xo)[node] = r;
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_copy_pdl(const double* __restrict__ x, double* __restrict__ xo) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int i = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 8 + threadIdx.y;
  if (i >= NX || j >= NY) return;
  const int node = i + NX * j;
  reinterpret_cast<double2*>(xo)[node] = __ldg(reinterpret_cast<const double2*>(x) + node);
}

// ---------------- variant C: direct loads, RY nodes per thread in y ----------
template <int RY, int MINB>
__global__ void __launch_bounds__(256, MINB) k_direct_ry(const __grid_constant__ KE ke, const double* __restrict__ x,
    const double* __restrict__ b, const double* __restrict__ dinv, const double* __restrict__ E,
    const uint8_t* __restrict__ mask, double w, double* __restrict__ xo) {
  const int i = blockIdx.x * 32 + threadIdx.x, j0 = (blockIdx.y * 8 + threadIdx.y) * RY;
  if (i >= NX || j0 >= NY) return;
  constexpr int R = RY + 2;
  double xs[R][3][2]; unsigned mk[R][3]; double ev[RY + 1][2];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int ii = i + c - 1, jj = j0 + r - 1;
      const bool in = ii >= 0 && ii < NX && jj >= 0 && jj < NY;
      const int n = in ? ii + NX * jj : 0;
      const double2 v = __ldg(reinterpret_cast<const double2*>(x) + n);
      xs[r][c][0] = v.x; xs[r][c][1] = v.y;
      mk[r][c] = in ? __ldg(mask + n) : 0u;
    }
#pragma unroll
  for (int r = 0; r <= RY; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int ex = i - 1 + c, ey = j0 - 1 + r;
      const bool in = ex >= 0 && ex < EXn && ey >= 0 && ey < EYn;
      ev[r][c] = in ? __ldg(E + ex + EXn * ey) : 0.0;
    }
  double2 bb[RY], dd[RY];
#pragma unroll
  for (int q = 0; q < RY; ++q) {
    const int jj = min(j0 + q, NY - 1);
    bb[q] = __ldg(reinterpret_cast<const double2*>(b) + i + NX * jj);
    dd[q] = __ldg(reinterpret_cast<const double2*>(dinv) + i + NX * jj);
  }
  double self[RY][2];
#pragma unroll
  for (int q = 0; q < RY; ++q) { self[q][0] = xs[q + 1][1][0]; self[q][1] = xs[q + 1][1][1]; }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (!(mk[r][c] & 1)) xs[r][c][0] = 0.0;
      if (!(mk[r][c] & 2)) xs[r][c][1] = 0.0;
    }
#pragma unroll
  for (int q = 0; q < RY; ++q) {
    if (j0 + q >= NY) break;
    double acc[2] = {0, 0};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int exo = e & 1, eyo = e >> 1;
      const int ln = corner_of(1 - exo, 1 - eyo);
      double t[2] = {0, 0};
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int rr = q + eyo + cy(m), cc = exo + cx(m);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int d = 0; d < 2; ++d) t[c] += ke.k[(ln * 2 + c) * 8 + m * 2 + d] * xs[rr][cc][d];
      }
      acc[0] += ev[q + eyo][exo] * t[0]; acc[1] += ev[q + eyo][exo] * t[1];
    }
    const unsigned mn = mk[q + 1][1];
    const double o0 = (mn & 1) ? acc[0] : self[q][0], o1 = (mn & 2) ? acc[1] : self[q][1];
    double2 r;
    r.x = self[q][0] + w * (dd[q].x * (bb[q].x - o0));
    r.y = self[q][1] + w * (dd[q].y * (bb[q].y - o1));
    reinterpret_cast<double2*>(xo)[i + NX * (j0 + q)] = r;
  }
}

// ---------------- variant A: smem tile (the library's current scheme) --------
constexpr int BX = 32, BY = 8, HX = BX + 2, HY = BY + 2, EX = BX + 1, EY = BY + 1;
__global__ void __launch_bounds__(256, 4) k_tiled(const __grid_constant__ KE ke, const double* __restrict__ x,
    const double* __restrict__ b, const double* __restrict__ dinv, const double* __restrict__ E,
    const uint8_t* __restrict__ mask, double w, double* __restrict__ xo) {
  __shared__ double2 xs_[HX * HY];
  __shared__ double es[EX * EY];
  __shared__ unsigned char ms[HX * HY];
  const int i0 = blockIdx.x * BX - 1, j0 = blockIdx.y * BY - 1;
  const int t0 = threadIdx.x + 32 * threadIdx.y;
  double2 v[2]; unsigned mk[2]; double ev[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int t = t0 + 256 * u, hx = t % HX, hy = t / HX, gi = i0 + hx, gj = j0 + hy;
    const bool in = t < HX * HY && gi >= 0 && gi < NX && gj >= 0 && gj < NY;
    const int n = in ? gi + NX * gj : 0;
    v[u] = in ? __ldg(reinterpret_cast<const double2*>(x) + n) : make_double2(0, 0);
    mk[u] = in ? __ldg(mask + n) : 0u;
    const int ex = t % EX, ey = t / EX, gex = i0 + ex, gey = j0 + ey;
    const bool ein = t < EX * EY && gex >= 0 && gex < EXn && gey >= 0 && gey < EYn;
    ev[u] = ein ? __ldg(E + gex + EXn * gey) : 0.0;
  }
  const int i = blockIdx.x * BX + threadIdx.x, j = blockIdx.y * BY + threadIdx.y;
  const bool active = i < NX && j < NY;
  const int node = active ? i + NX * j : 0;
  const double2 bb = __ldg(reinterpret_cast<const double2*>(b) + node);
  const double2 dd = __ldg(reinterpret_cast<const double2*>(dinv) + node);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int t = t0 + 256 * u;
    if (t < HX * HY) { xs_[t] = v[u]; ms[t] = (unsigned char)mk[u]; }
    if (t < EX * EY) es[t] = ev[u];
  }
  __syncthreads();
  if (!active) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  double xs[9][2]; double self[2];
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const int h = (tx + s % 3) + HX * (ty + s / 3);
    const double2 q = xs_[h]; const unsigned m = ms[h];
    if (s == 4) { self[0] = q.x; self[1] = q.y; }
    xs[s][0] = (m & 1) ? q.x : 0.0; xs[s][1] = (m & 2) ? q.y : 0.0;
  }
  double acc[2] = {0, 0};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int exo = e & 1, eyo = e >> 1;
    const int ln = corner_of(1 - exo, 1 - eyo);
    double t[2] = {0, 0};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int s = (exo + cx(m)) + 3 * (eyo + cy(m));
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int d = 0; d < 2; ++d) t[c] += ke.k[(ln * 2 + c) * 8 + m * 2 + d] * xs[s][d];
    }
    const double Ee = es[(tx + exo) + EX * (ty + eyo)];
    acc[0] += Ee * t[0]; acc[1] += Ee * t[1];
  }
  const unsigned mn = ms[(tx + 1) + HX * (ty + 1)];
  const double o0 = (mn & 1) ? acc[0] : self[0], o1 = (mn & 2) ? acc[1] : self[1];
  double2 r;
  r.x = self[0] + w * (dd.x * (bb.x - o0));
  r.y = self[1] + w * (dd.y * (bb.y - o1));
  reinterpret_cast<double2*>(xo)[node] = r;
}

static cudaStream_t g_s;
// reps launches captured into one CUDA graph (no host launch overhead in the timing)
template <class F>
float timeit(F f, int reps) {
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(g_s, cudaStreamCaptureModeGlobal));
  for (int r = 0; r < reps; ++r) f();
  CK(cudaStreamEndCapture(g_s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaGraphLaunch(ge, g_s));
  cudaEventRecord(a, g_s);
  CK(cudaGraphLaunch(ge, g_s));
  cudaEventRecord(b, g_s); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  return 1e3f * ms / reps;
}

int main() {
  const int nn = NX * NY, nd = 2 * nn, ne = EXn * EYn;
  CK(cudaStreamCreateWithFlags(&g_s, cudaStreamNonBlocking));
  KE ke;
  for (int a = 0; a < 8; ++a) for (int c = 0; c < 8; ++c) ke.k[a * 8 + c] = (a == c ? 1.0 : 0.0) + 0.01 * ((a * 7 + c * 3) % 11) * (a == c ? 0 : 1) + 0.01 * ((c * 7 + a * 3) % 11);
  std::vector<double> hx(nd), hb(nd), hd(nd), he(ne);
  std::vector<uint8_t> hm(nn);
  srand(1);
  for (int i = 0; i < nd; ++i) { hx[i] = rand() / (double)RAND_MAX; hb[i] = rand() / (double)RAND_MAX; hd[i] = 0.5 + rand() / (double)RAND_MAX; }
  for (int i = 0; i < ne; ++i) he[i] = rand() % 2 ? 1.0 : 1e-9;
  for (int i = 0; i < nn; ++i) hm[i] = (i % NX == 0) ? 2 : 3;
  double *x, *b, *d, *E, *o1, *o2, *o3; uint8_t* m;
  CK(cudaMalloc(&x, nd * 8)); CK(cudaMalloc(&b, nd * 8)); CK(cudaMalloc(&d, nd * 8)); CK(cudaMalloc(&E, ne * 8));
  CK(cudaMalloc(&o1, nd * 8)); CK(cudaMalloc(&o2, nd * 8)); CK(cudaMalloc(&o3, nd * 8)); CK(cudaMalloc(&m, nn));
  cudaMemcpy(x, hx.data(), nd * 8, cudaMemcpyHostToDevice); cudaMemcpy(b, hb.data(), nd * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d, hd.data(), nd * 8, cudaMemcpyHostToDevice); cudaMemcpy(E, he.data(), ne * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(m, hm.data(), nn, cudaMemcpyHostToDevice);
  const double bytes = nd * 32.0 + ne * 8.0 + nn;
  dim3 blk(32, 8), g1((NX + 31) / 32, (NY + 7) / 8);
  const int reps = 200;
  auto report = [&](const char* name, float us, double* out) {
    std::vector<double> h(nd), r(nd);
    cudaMemcpy(h.data(), out, nd * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(r.data(), o1, nd * 8, cudaMemcpyDeviceToHost);
    double md = 0; for (int i = 0; i < nd; ++i) md = fmax(md, fabs(h[i] - r[i]));
    printf("%-28s %7.2f us  %7.0f GB/s  maxdiff %.2e\n", name, us, bytes / us / 1e3, md);
  };
  float t;
  t = timeit([&] { k_tiled<<<g1, blk, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o1); }, reps); report("A tiled smem", t, o1);
  t = timeit([&] { k_direct<4><<<g1, blk, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o2); }, reps); report("B direct minb4", t, o2);
  t = timeit([&] { k_direct<2><<<g1, blk, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o2); }, reps); report("B direct minb2", t, o2);
  t = timeit([&] { k_direct<1><<<g1, blk, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o2); }, reps); report("B direct minb1", t, o2);
  dim3 g2((NX + 31) / 32, (NY + 15) / 16), g4((NX + 31) / 32, (NY + 31) / 32);
  t = timeit([&] { k_direct_ry<2, 2><<<g2, blk, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o3); }, reps); report("C direct ry2 minb2", t, o3);
  t = timeit([&] { k_direct_ry<2, 1><<<g2, blk, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o3); }, reps); report("C direct ry2 minb1", t, o3);
  t = timeit([&] { k_direct_ry<4, 1><<<g4, blk, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o3); }, reps); report("C direct ry4 minb1", t, o3);
  t = timeit([&] { k_direct_ry<4, 2><<<g4, blk, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o3); }, reps); report("C direct ry4 minb2", t, o3);
  // plain copy roofline for reference: read 3 vectors, write 1
  t = timeit([&] { cudaMemcpyAsync(o2, x, nd * 8, cudaMemcpyDeviceToDevice, g_s); }, reps);
  printf("memcpy %d B: %.2f us (%.0f GB/s)\n", nd * 8, t, 2.0 * nd * 8 / t / 1e3);
  {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = g1; cfg.blockDim = blk; cfg.stream = g_s;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 0;
    t = timeit([&] { CK(cudaLaunchKernelEx(&cfg, k_copy_pdl<4>, (const double*)x, o2)); }, reps);
    printf("node copy kernel, no PDL: %.2f us\n", t);
    cfg.numAttrs = 1;
    t = timeit([&] { CK(cudaLaunchKernelEx(&cfg, k_copy_pdl<4>, (const double*)x, o2)); }, reps);
    printf("node copy kernel, PDL: %.2f us\n", t);
    cfg.gridDim = dim3(1); cfg.blockDim = dim3(32); cfg.numAttrs = 0;
    t = timeit([&] { CK(cudaLaunchKernelEx(&cfg, k_copy_pdl<4>, (const double*)x, o2)); }, reps);
    printf("1-block, no PDL: %.2f us\n", t);
    cfg.numAttrs = 1;
    t = timeit([&] { CK(cudaLaunchKernelEx(&cfg, k_copy_pdl<4>, (const double*)x, o2)); }, reps);
    printf("1-block, PDL: %.2f us\n", t);
  }
  // empty-ish kernel floor
  t = timeit([&] { k_direct<4><<<1, 32, 0, g_s>>>(ke, x, b, d, E, m, 0.6, o2); }, reps);
  printf("1-block launch floor: %.2f us\n", t);
  return 0;
}
