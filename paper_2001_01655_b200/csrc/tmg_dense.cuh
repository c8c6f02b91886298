// Coarsest-level direct solve (reference: splu of the coarsest operator at build
// time, multigrid.py:256).  On the B200 the coarse operator is factorised once
// at setup -- blocked Cholesky on the FP64 tensor pipe, the explicit inverse
// formed from the factor (tmg_chol.cuh) -- and every V-cycle then applies the
// inverse as one bandwidth-bound GEMV instead of two latency-bound triangular
// solves.  TMG_COARSE=gj selects the blocked Gauss-Jordan inverse below (the
// round-1 path: NB-column pivot blocks, rank-NB DMMA trailing updates), kept
// as the measured A/B baseline.
#pragma once
#include "tmg_common.cuh"
#include "tmg_chol.cuh"

namespace tmg {

constexpr int GJ_NB = 32;

// In-place Gauss-Jordan of the kb x kb pivot block; writes D = A_KK^-1.
// Thread (i, j) keeps M[i][j] in a register: M[i][p] comes from lane p of the
// same warp (shuffle), the pivot row from a double-buffered shared row written
// by warp p at the end of step p-1 -- one barrier per step instead of two, same
// arithmetic per entry.
__global__ void __launch_bounds__(1024) k_gj_pivot(const double* __restrict__ A, long long n, long long k0, int kb,
                                                   double* __restrict__ D, unsigned* __restrict__ bad) {
  TMG_PDL_ENTRY;
  __shared__ double prow[2][GJ_NB];
  const int i = threadIdx.y, j = threadIdx.x;
  const bool in = i < kb && j < kb;
  double m = in ? A[(k0 + i) * n + k0 + j] : 0.0;
  if (i == 0) prow[0][j] = m;
  __syncthreads();
  for (int p = 0; p < kb; ++p) {
    const double mpj = prow[p & 1][j];
    double piv = prow[p & 1][p];
    const double mip = __shfl_sync(0xffffffffu, m, p);
    if (!(piv > 0.0)) {
      if (i == 0 && j == 0) atomicOr(bad, 1u);
      piv = 1.0;
    }
    const double d = 1.0 / piv;
    if (in) {
      if (i == p && j == p) m = d;
      else if (i == p) m = mpj * d;
      else if (j == p) m = -mip * d;
      else m = m - mip * mpj * d;
    }
    if (i == p + 1) prow[(p + 1) & 1][j] = m;
    __syncthreads();
  }
  if (in) D[i * GJ_NB + j] = m;
}

// RowP[r][j] = sum_c D[r][c] A[k0+c][j]  (all j);  ColP[c][i] = A[i][k0+c]
// (column-major copy of the pivot columns: the update kernels stage it coalesced).
// blockIdx.y picks GJ_PANEL_R rows r of D (and the same columns c of the ColP
// copy): n/128 x 8 blocks instead of n/256, so the 2562-wide config-1 panel
// fills the SMs (measured 15.8 us on 11 blocks).  Each sum keeps the c order.
constexpr int GJ_PANEL_R = 4, GJ_PANEL_TPB = 128;
__global__ void __launch_bounds__(GJ_PANEL_TPB) k_gj_panels(const double* __restrict__ A, long long n, long long k0,
                                                            int kb, const double* __restrict__ D,
                                                            double* __restrict__ RowP, double* __restrict__ ColP) {
  TMG_PDL_ENTRY;
  __shared__ double Ds[GJ_PANEL_R * GJ_NB];
  const int r0 = blockIdx.y * GJ_PANEL_R;
  for (int t = threadIdx.x; t < GJ_PANEL_R * GJ_NB; t += blockDim.x) Ds[t] = D[r0 * GJ_NB + t];
  __syncthreads();
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double col[GJ_NB];
#pragma unroll
  for (int c = 0; c < GJ_NB; ++c) col[c] = c < kb ? A[(k0 + c) * n + j] : 0.0;
#pragma unroll
  for (int q = 0; q < GJ_PANEL_R; ++q) {
    const int r = r0 + q;
    if (r >= kb) break;
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < GJ_NB; ++c) s += Ds[q * GJ_NB + c] * col[c];
    RowP[r * n + j] = s;
  }
#pragma unroll
  for (int q = 0; q < GJ_PANEL_R; ++q) {
    const int c = r0 + q;
    if (c < kb) ColP[c * n + j] = A[j * n + k0 + c];
  }
}

// 64x64 output tile per block, 256 threads x (4x4) outputs.
__global__ void __launch_bounds__(256) k_gj_update(double* __restrict__ A, long long n, long long k0, int kb,
                                                   const double* __restrict__ D, const double* __restrict__ RowP,
                                                   const double* __restrict__ ColP) {
  TMG_PDL_ENTRY;
  __shared__ double Cs[GJ_NB][64 + 1];  // Cs[c][ii] = ColP[c][i0+ii]
  __shared__ double Rs[GJ_NB][64 + 1];  // Rs[c][jj] = RowP[c][j0+jj]
  __shared__ double Ds[GJ_NB][GJ_NB + 1];
  const long long i0 = blockIdx.y * 64LL, j0 = blockIdx.x * 64LL;
  for (int t = threadIdx.x; t < GJ_NB * 64; t += blockDim.x) {
    const int c = t / 64, q = t % 64;
    const long long gi = i0 + q, gj = j0 + q;
    Cs[c][q] = (c < kb && gi < n) ? ColP[c * n + gi] : 0.0;
    Rs[c][q] = (c < kb && gj < n) ? RowP[c * n + gj] : 0.0;
  }
  for (int t = threadIdx.x; t < GJ_NB * GJ_NB; t += blockDim.x) Ds[t / GJ_NB][t % GJ_NB] = D[t];
  __syncthreads();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int c = 0; c < kb; ++c) {
    double cv[4], rv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) cv[a] = Cs[c][ty + 16 * a];
#pragma unroll
    for (int b = 0; b < 4; ++b) rv[b] = Rs[c][tx + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] += cv[a] * rv[b];
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const long long gi = i0 + ty + 16 * a;
    if (gi >= n) continue;
    const bool iK = gi >= k0 && gi < k0 + kb;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const long long gj = j0 + tx + 16 * b;
      if (gj >= n) continue;
      const bool jK = gj >= k0 && gj < k0 + kb;
      double* dst = &A[gi * n + gj];
      if (!iK && !jK) {
        *dst -= acc[a][b];
      } else if (iK && !jK) {
        *dst = Rs[gi - k0][tx + 16 * b];
      } else if (!iK && jK) {
        double s = 0.0;
        for (int c = 0; c < kb; ++c) s += Cs[c][ty + 16 * a] * Ds[c][gj - k0];
        *dst = -s;
      } else {
        *dst = Ds[gi - k0][gj - k0];
      }
    }
  }
}

// The same rank-kb update on the FP64 tensor pipe: DMMA m8n8k4 (mma.sync .f64).
// 64x64 output tile per block; warp w owns a 16x32 sub-tile = 2x4 MMA tiles.
// Fragments (PTX m8n8k4 .f64, row.col): lane l = 4g + t holds A[g][t], B[t][g]
// and C[g][2t..2t+1] of its 8x8 tile.  Operands come from the same shared-memory
// panels as k_gj_update; only the pivot rows/columns take the scalar path.
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(256) k_gj_update_mma(double* __restrict__ A, long long n, long long k0, int kb,
                                                       const double* __restrict__ D,
                                                       const double* __restrict__ RowP,
                                                       const double* __restrict__ ColP) {
  TMG_PDL_ENTRY;
  // row stride 68 doubles (4 mod 16): the fragment loads below (lane 4g+t reads
  // [c+t][base+g]) hit 16 distinct bank pairs per half-warp
  __shared__ double Cs[GJ_NB][64 + 4];  // Cs[c][ii] = ColP[c][i0+ii]
  __shared__ double Rs[GJ_NB][64 + 4];  // Rs[c][jj] = RowP[c][j0+jj]
  __shared__ double Ds[GJ_NB][GJ_NB + 1];
  const long long i0 = blockIdx.y * 64LL, j0 = blockIdx.x * 64LL;
  for (int t = threadIdx.x; t < GJ_NB * 64; t += blockDim.x) {
    const int c = t / 64, q = t % 64;
    const long long gi = i0 + q, gj = j0 + q;
    Cs[c][q] = (c < kb && gi < n) ? ColP[c * n + gi] : 0.0;
    Rs[c][q] = (c < kb && gj < n) ? RowP[c * n + gj] : 0.0;
  }
  for (int t = threadIdx.x; t < GJ_NB * GJ_NB; t += blockDim.x) Ds[t / GJ_NB][t % GJ_NB] = D[t];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 32;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int kr = (kb + 3) & ~3;  // rows c >= kb of the panels are zero
#pragma unroll 4
  for (int c = 0; c < kr; c += 4) {
    double av[2], bv[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) av[a] = Cs[c + tq][r0 + a * 8 + g];
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = Rs[c + tq][c0 + b * 8 + g];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b], av[a], bv[b]);
  }
  const bool vec = (n & 1) == 0;  // rows 16-byte aligned: RMW the two outputs of a lane as one double2
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int ii = r0 + a * 8 + g;
    const long long gi = i0 + ii;
    if (gi >= n) continue;
    const bool iK = gi >= k0 && gi < k0 + kb;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int jj0 = c0 + b * 8 + 2 * tq;
      const long long gj0 = j0 + jj0;
      const bool plain = vec && !iK && gj0 + 1 < n && !(gj0 + 1 >= k0 && gj0 < k0 + kb);
      if (plain) {
        double2* dst = reinterpret_cast<double2*>(&A[gi * n + gj0]);
        double2 v = *dst;
        v.x -= acc[a][b][0];
        v.y -= acc[a][b][1];
        *dst = v;
        continue;
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jj = jj0 + e;
        const long long gj = j0 + jj;
        if (gj >= n) continue;
        const bool jK = gj >= k0 && gj < k0 + kb;
        double* dst = &A[gi * n + gj];
        if (!iK && !jK) {
          *dst -= acc[a][b][e];
        } else if (iK && !jK) {
          *dst = Rs[gi - k0][jj];
        } else if (!iK && jK) {
          double sacc = 0.0;
          for (int c = 0; c < kb; ++c) sacc += Cs[c][ii] * Ds[c][gj - k0];
          *dst = -sacc;
        } else {
          *dst = Ds[gi - k0][gj - k0];
        }
      }
    }
  }
}

// y = Ainv b: one warp per row, coalesced row reads.
__global__ void __launch_bounds__(256) k_gemv_rows(const double* __restrict__ A, long long n,
                                                   const double* __restrict__ b, double* __restrict__ y) {
  TMG_PDL_ENTRY;
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* a = A + row * n;
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long j = lane;
  for (; j + 7 * 32 < n; j += 8 * 32) {  // 8 independent row loads in flight per lane
    double av[8], bv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) av[u] = __ldg(a + j + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) bv[u] = __ldg(b + j + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) s[u] += av[u] * bv[u];
  }
  for (; j < n; j += 32) s[0] += a[j] * b[j];
  double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  t = warp_sum(t);
  if (lane == 0) y[row] = t;
}
// Even n (rows 16-byte aligned): one row per block of S warps (split-K), 128-bit
// loads; S x the bytes in flight of a warp-per-row kernel (2562 rows leave only
// ~17 warps per SM otherwise, the coarsest inverse is 52 MB on config 1).  The
// S partial sums are combined in a fixed order (deterministic).
template <int S>
__global__ void __launch_bounds__(32 * S) k_gemv_split(const double* __restrict__ A, long long n,
                                                      const double* __restrict__ b, double* __restrict__ y) {
  TMG_PDL_ENTRY;
  __shared__ double part[S];
  const long long row = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double2* a = reinterpret_cast<const double2*>(A + row * n);
  const double2* bb = reinterpret_cast<const double2*>(b);
  const long long n2 = n >> 1;
  double s[4] = {0, 0, 0, 0};
  long long j = threadIdx.x;
  constexpr int T = 32 * S;
  for (; j + 3 * T < n2; j += 4 * T) {
    double2 av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) av[u] = __ldg(a + j + T * u);
#pragma unroll
    for (int u = 0; u < 4; ++u) bv[u] = __ldg(bb + j + T * u);
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] += av[u].x * bv[u].x + av[u].y * bv[u].y;
  }
  for (int u = 0; j < n2; j += T, ++u) {
    const double2 av = __ldg(a + j), bv = __ldg(bb + j);
    s[u & 3] += av.x * bv.x + av.y * bv.y;
  }
  double t = (s[0] + s[1]) + (s[2] + s[3]);
  t = warp_sum(t);
  if (lane == 0) part[w] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
#pragma unroll
    for (int q = 0; q < S; ++q) r += part[q];
    y[row] = r;
  }
}

// TMG_DENSE_MMA=0 selects the CUDA-core update (A/B switch and parity check).
inline bool dense_mma() {
  static const bool on = [] {
    const char* e = std::getenv("TMG_DENSE_MMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Dense SPD inverse on the device (setup; stream-ordered, no host sync): Cholesky
// (default) or Gauss-Jordan (TMG_COARSE=gj).
struct DenseInverse {
  long long n = 0;
  DevBuf<double> A;  // holds the inverse after build()
  DevBuf<double> D, RowP, ColP;
  DevBuf<unsigned> bad;
  static bool use_gj() {
    static const bool gj = [] {
      const char* e = std::getenv("TMG_COARSE");
      return e && e[0] == 'g';
    }();
    return gj;
  }
  void build(cudaStream_t s) {
    if (!use_gj()) {
      bad.alloc(1, s);
      bad.zero(s);
      cholesky_inverse(A.get(), n, bad.get(), s);
      return;
    }
    D.alloc(GJ_NB * GJ_NB, s);
    RowP.alloc((size_t)GJ_NB * n, s);
    ColP.alloc((size_t)GJ_NB * n, s);
    bad.alloc(1, s);
    bad.zero(s);
    const unsigned tiles = (unsigned)((n + 63) / 64);
    for (long long k0 = 0; k0 < n; k0 += GJ_NB) {
      const int kb = (int)std::min<long long>(GJ_NB, n - k0);
      launch(k_gj_pivot, 1, dim3(GJ_NB, GJ_NB), 0, s, A.get(), n, k0, kb, D.get(), bad.get()); ::tmg::note_launch();
      launch(k_gj_panels, dim3((unsigned)((n + GJ_PANEL_TPB - 1) / GJ_PANEL_TPB), GJ_NB / GJ_PANEL_R), GJ_PANEL_TPB, 0, s, A.get(), n, k0, kb, D.get(), RowP.get(), ColP.get()); ::tmg::note_launch();
      launch(dense_mma() ? k_gj_update_mma : k_gj_update, dim3(tiles, tiles), 256, 0, s, A.get(), n, k0, kb, D.get(),
             RowP.get(), ColP.get());
      ::tmg::note_launch();
    }
    TMG_CUDA(cudaGetLastError());
    RowP.release();
    ColP.release();
    D.release();
  }
  void apply(const double* b, double* y, cudaStream_t s) const {
    // measured on config 1's 2562-row inverse: split-K 4 warps 9.3 us, warp per
    // row 11.5 us, 8 warps 12.7 us
    if ((n & 1) == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0)
      launch(k_gemv_split<4>, (unsigned)n, 128, 0, s, A.get(), n, b, y);
    else
      launch(k_gemv_rows, grid_for(n * 32), 256, 0, s, A.get(), n, b, y);
    ::tmg::note_launch();
  }
};

}  // namespace tmg
