// Vector kernels (reductions, scalings, Lanczos pieces) and the device stiffness
// operator K(rho) shared by every hierarchy kind.
#pragma once
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <memory>

#include "tmg_dense.cuh"
#include "tmg_ke.h"
#include "tmg_ops.cuh"

namespace tmg {

enum SmootherKind { SM_JACOBI = 0, SM_BLOCK_JACOBI = 1, SM_CHEBYSHEV = 2, SM_SOR_CHEBYSHEV = 3, SM_SOR_GMRES = 4 };
inline bool sor_kind(int k) { return k == SM_SOR_CHEBYSHEV || k == SM_SOR_GMRES; }
inline bool cheb_kind(int k) { return k == SM_CHEBYSHEV || k == SM_SOR_CHEBYSHEV; }

struct SmootherCfg {
  int kind = SM_JACOBI;
  double weight = 0.5;
  int degree = 2;
  int lanczos_steps = 10;
  uint64_t seed = 0;
  double safeguard = 0.0;  // >0: Jacobi weight capped at safeguard / lambda_hat (Lanczos)
  const double* power_start = nullptr;  // sor_chebyshev: device start vector (>= level-0 dofs)
};

// ----------------------------------------------------------------------------
// small vector kernels
// ----------------------------------------------------------------------------
// Reduction kernels run on a small grid (RED_BLOCKS) with 4 independent loads in
// flight per thread, so the last-block combine reads few partials.
#ifndef TMG_RED_BLOCKS
#define TMG_RED_BLOCKS 296
#endif
constexpr unsigned RED_BLOCKS = TMG_RED_BLOCKS;  // 2 per SM
inline unsigned red_grid(long long n) { return std::min<unsigned>(grid_for(n), RED_BLOCKS); }

__global__ void __launch_bounds__(TPB) k_dot(const double* __restrict__ a, const double* __restrict__ b, long long n,
                                             Red red) {
  TMG_PDL_ENTRY;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const double a0 = __ldg(a + i), a1 = __ldg(a + i + stride), a2 = __ldg(a + i + 2 * stride),
                 a3 = __ldg(a + i + 3 * stride);
    const double b0 = __ldg(b + i), b1 = __ldg(b + i + stride), b2 = __ldg(b + i + 2 * stride),
                 b3 = __ldg(b + i + 3 * stride);
    s0 += a0 * b0; s1 += a1 * b1; s2 += a2 * b2; s3 += a3 * b3;
  }
  for (; i < n; i += stride) s0 += a[i] * b[i];
  grid_reduce((s0 + s1) + (s2 + s3), red);
}
__global__ void k_scale_vec(const double* __restrict__ b, const double* __restrict__ d, const double* __restrict__ wp,
                            double* __restrict__ x, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) x[i] = *wp * (d[i] * b[i]);
}
template <int DIM>
__global__ void k_bscale_vec(const double* __restrict__ b, const double* __restrict__ binv, const double* __restrict__ wp,
                             double* __restrict__ x, long long nnodes) {
  TMG_PDL_ENTRY;
  const long long node = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (node >= nnodes) return;
  const double w = *wp;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < DIM; ++c) s += binv[node * DIM * DIM + a * DIM + c] * b[node * DIM + c];
    x[node * DIM + a] = w * s;
  }
}
__global__ void k_recip(const double* __restrict__ d, double* __restrict__ dinv, double* __restrict__ dsq, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  dinv[i] = 1.0 / d[i];
  if (dsq) dsq[i] = sqrt(1.0 / d[i]);
}
// splitmix64 start vector, bit-identical to oracle.splitmix_uniform
__global__ void k_splitmix(double* __restrict__ v, long long n, unsigned long long seed) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long G = 0x9E3779B97F4A7C15ULL;
  unsigned long long z = seed * G + (unsigned long long)(i + 1) * G;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  v[i] = (double)(z >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}
__global__ void k_div_sqrt(double* __restrict__ v, const double* __restrict__ s2, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = v[i] / sqrt(*s2);
}
// w -= a v + b vprev  (b from beta2 slot j-1 or 0)
__global__ void k_lz_orth(double* __restrict__ w, const double* __restrict__ v, const double* __restrict__ vp,
                          const double* __restrict__ alpha, const double* __restrict__ beta2, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = *alpha;
  const double b = beta2 ? sqrt(*beta2) : 0.0;
  w[i] = b != 0.0 ? w[i] - a * v[i] - b * vp[i] : w[i] - a * v[i];
}
__global__ void k_lz_next(double* __restrict__ v, double* __restrict__ vp, const double* __restrict__ w,
                          const double* __restrict__ beta2, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  vp[i] = v[i];
  v[i] = w[i] / sqrt(*beta2);
}
// Largest eigenvalue of the Lanczos tridiagonal by Sturm bisection, then the
// Chebyshev step coefficients on [0.1, 1.1] * lambda (multigrid.py:129-149).
// With wout: the safeguarded Jacobi weight min(w0, sg / lambda) instead.
__global__ void k_lz_finish(const double* __restrict__ alpha, const double* __restrict__ beta2, int steps,
                            int degree, double* __restrict__ coef, double* __restrict__ lmax_out, double w0,
                            double sg, double* __restrict__ wout) {
  TMG_PDL_ENTRY;
  int m = steps;
  for (int j = 0; j < steps; ++j)
    if (!(sqrt(beta2[j]) > 1e-300)) { m = j + 1; break; }
  double lo = 1e300, hi = -1e300;
  for (int j = 0; j < m; ++j) {
    const double bl = j > 0 ? sqrt(beta2[j - 1]) : 0.0, br = j < m - 1 ? sqrt(beta2[j]) : 0.0;
    lo = fmin(lo, alpha[j] - bl - br);
    hi = fmax(hi, alpha[j] + bl + br);
  }
  for (int it = 0; it < 200; ++it) {  // count of eigenvalues < x via LDL^T pivots
    const double x = 0.5 * (lo + hi);
    if (x == lo || x == hi) break;
    int cnt = 0;
    double q = 1.0;
    for (int j = 0; j < m; ++j) {
      const double b2 = j > 0 ? beta2[j - 1] : 0.0;
      q = (alpha[j] - x) - (j > 0 ? b2 / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0.0) ++cnt;
    }
    if (cnt == m) hi = x; else lo = x;
  }
  const double lam = hi;
  *lmax_out = lam;
  if (wout) *wout = fmin(w0, sg / lam);
  if (!coef) return;
  const double a = 0.1 * lam, b = 1.1 * lam, theta = 0.5 * (b + a), delta = 0.5 * (b - a);
  double al = 0.0, be = 0.0;
  for (int i = 0; i < degree; ++i) {
    if (i == 0) { al = 1.0 / theta; be = 0.0; }
    else { be = (delta * al / 2.0) * (delta * al / 2.0); al = 1.0 / (theta - be / al); }
    coef[2 * i] = al;
    coef[2 * i + 1] = be;
  }
}

// ----------------------------------------------------------------------------
// the stiffness operator K(rho) (mesh.py:327)
// ----------------------------------------------------------------------------
struct Operator {
  int dim = 2;
  Lat L{};
  int ne[3] = {1, 1, 1};
  double h[3] = {1, 1, 1};
  double nu = 0.3;
  long long nelem = 0, ndof = 0;
  DevBuf<double> E, ke;
  DevBuf<uint8_t> mask;
  std::vector<double> ke_host;
  std::vector<double> keh_host;  // 3D: KE in the reflection-character basis (tmg_fine3h.cuh)
  template <int DIM>
  FineOp<DIM> fine() const {
    FineOp<DIM> o;
    o.L = L;
    for (int d = 0; d < 3; ++d) o.ne[d] = ne[d];
    o.E = E.get();
    o.mask = mask.get();
    std::memcpy(o.ke, ke_host.data(), sizeof(o.ke));
    if constexpr (DIM == 3) std::memcpy(o.keh, keh_host.data(), sizeof(o.keh));
    return o;
  }
};
}  // namespace tmg
