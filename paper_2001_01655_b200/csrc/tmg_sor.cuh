// SOR smoothers of the reference (multigrid.py:97-176) and block Jacobi on
// algebraic levels (multigrid.py:64), device kernels.
//
// The reference's SOR "sweep" is a sparse lower-triangular solve
// z = tril(A)^-1 v (scipy spsolve_triangular, omega = 1: forward Gauss-Seidel).
// Here it runs as a synchronisation-free block-row solve on the level's BSR
// form (lattice levels are converted once at setup): one warp per block row,
// rows handed out by an atomic ticket in a topological order (level sets of the
// dependency DAG, computed at setup), each warp spins on the ready flags of the
// rows it depends on, forms rhs = v_I - sum_{J<I} A_IJ z_J, then forward-
// substitutes with the lower triangle of its diagonal block (= scalar Gauss-
// Seidel in dof order, dofs being block-contiguous).  Flags carry the epoch of
// the solve that set them, so no reset pass is needed between solves.
// Deadlock freedom: a ticket is only drawn by a running warp, and every
// dependency of a row precedes it in the ticket order.
#pragma once
#include "tmg_bsr.cuh"

namespace tmg {

struct SorView {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const double* __restrict__ val;
  const int* __restrict__ diagpos;  // position of the diagonal block of each row
  const int* __restrict__ order;    // ticket -> block row (topological)
  int nrows;
  int* flag;  // per block row: epoch of the last solve that finished it
  int* ctl;   // [0] epoch, [1] ticket counter
  int sleep_ns;  // poll back-off cap (0: spin)
  int acquire;   // 1: acquire once per observed dependency (z is read through L2 either way)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Polls use relaxed loads: an acquire load also invalidates the SM's L1, and
// with hundreds of polling warps per SM that evicts every row's prefetched
// blocks.  Only the final, successful observation is an acquire.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// new epoch, ticket counter back to zero (one thread, before every solve)
__global__ void k_sor_prep(int* ctl) {
  TMG_PDL_ENTRY;
  ctl[0] += 1;
  ctl[1] = 0;
}

constexpr int SOR_TPB = 256;

template <int R>
__global__ void __launch_bounds__(SOR_TPB) k_sor_solve(SorView S, const double* __restrict__ v, double* z) {
  TMG_PDL_ENTRY;
  // Everything a row needs that does not depend on other rows (its right-hand
  // side, diagonal block and, for R <= 3, its lower blocks) is loaded BEFORE the
  // row waits on its dependencies, so a dependency hop costs one flag
  // observation + one z load + the arithmetic + one release store.
  constexpr bool PRE = R <= 3;
  const int lane = threadIdx.x & 31;
  const int epoch = *(volatile int*)S.ctl;
  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(S.ctl + 1, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= S.nrows) return;
    const int row = S.order[t];
    const int beg = S.rowptr[row], dp = S.diagpos[row];
    double D[PRE ? R * R : 1], vr[R];
    if (lane == 0) {
#pragma unroll
      for (int a = 0; a < R; ++a) vr[a] = v[(long long)row * R + a];
      if constexpr (PRE) {
#pragma unroll
        for (int q = 0; q < R * R; ++q) D[q] = __ldg(S.val + (long long)dp * R * R + q);
      }
    }
    double acc[R];
#pragma unroll
    for (int a = 0; a < R; ++a) acc[a] = 0.0;
    for (int p = beg + lane; p < dp; p += 32) {
      const int j = S.col[p];
      const double* blk = S.val + (long long)p * R * R;
      double bv[PRE ? R * R : 1];
      if constexpr (PRE) {
#pragma unroll
        for (int q = 0; q < R * R; ++q) bv[q] = __ldg(blk + q);
      }
      if (ld_relaxed(S.flag + j) != epoch) {
        // optional back-off: many spinning warps can saturate the L2 with polls
        unsigned ns = 8;
        do {
          if (S.sleep_ns) {
            __nanosleep(ns);
            ns = ns < (unsigned)S.sleep_ns ? 2 * ns : ns;
          }
        } while (ld_relaxed(S.flag + j) != epoch);
      }
      if (S.acquire) (void)ld_acquire(S.flag + j);
      double zj[R];
#pragma unroll
      for (int b = 0; b < R; ++b) zj[b] = __ldcg(z + (long long)j * R + b);
#pragma unroll
      for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < R; ++b) acc[a] += (PRE ? bv[a * R + b] : __ldg(blk + a * R + b)) * zj[b];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int a = 0; a < R; ++a) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], off);
    if (lane == 0) {
      const double* Dg = S.val + (long long)dp * R * R;
      double zi[R];
#pragma unroll
      for (int a = 0; a < R; ++a) {
        double s = vr[a] - acc[a];
#pragma unroll
        for (int b = 0; b < a; ++b) s -= (PRE ? D[a * R + b] : Dg[a * R + b]) * zi[b];
        zi[a] = s / (PRE ? D[a * R + a] : Dg[a * R + a]);
        z[(long long)row * R + a] = zi[a];
      }
      st_release(S.flag + row, epoch);
    }
    __syncwarp();
  }
}

// diagonal-block position of every block row; bad |= 4 for a zero diagonal entry
template <int R>
__global__ void k_sor_diagpos(BsrView<R, R> A, int* __restrict__ diagpos, unsigned* __restrict__ bad) {
  TMG_PDL_ENTRY;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  int dp = -1;
  for (int p = A.rowptr[row]; p < A.rowptr[row + 1]; ++p)
    if (A.col[p] == row) dp = p;
  diagpos[row] = dp;
  bool ok = dp >= 0;
  if (ok)
    for (int a = 0; a < R; ++a) ok = ok && A.val[(long long)dp * R * R + a * R + a] != 0.0;
  if (!ok) atomicOr(bad, 4u);
}

// ----------------------------------------------------------------------------
// SOR-Chebyshev pieces
// ----------------------------------------------------------------------------
// Chebyshev step coefficients on [0.1, 1.1] * lambda, lambda = ||w|| of the last
// power step (multigrid.py:120-149).
__global__ void k_sor_cheb_coef(const double* __restrict__ w2, int degree, double* __restrict__ coef,
                                double* __restrict__ lmax) {
  TMG_PDL_ENTRY;
  const double lam = sqrt(*w2);
  *lmax = lam;
  const double lo = 0.1 * lam, hi = 1.1 * lam, d = (hi + lo) / 2.0, c = (hi - lo) / 2.0;
  double al = 0.0, be = 0.0;
  for (int i = 0; i < degree; ++i) {
    if (i == 0) { al = 1.0 / d; be = 0.0; }
    else { be = (c * al / 2.0) * (c * al / 2.0); al = 1.0 / (d - be / al); }
    coef[2 * i] = al;
    coef[2 * i + 1] = be;
  }
}

// ----------------------------------------------------------------------------
// SOR-GMRES smoother: per pass one FGMRES cycle of m = inner_iterations steps,
// right-preconditioned by the SOR solve (multigrid.py:153-170 calls
// fgmres_solve with rtol 1e-14, max_iterations = restart = m).  Vector work is
// done by the usual kernels; the Givens / least-squares bookkeeping of
// krylov.py:96-125 runs in one thread on a per-level scalar block g:
// ----------------------------------------------------------------------------
constexpr double GM_BREAKDOWN = 1e-14;  // krylov.py:13 BREAKDOWN_TOL
constexpr double GM_RTOL = 1e-14;       // multigrid.py:164
struct GmLayout {                       // offsets into g (doubles)
  int M;
  __host__ __device__ int bb() const { return 0; }   // b.b
  __host__ __device__ int rr() const { return 1; }   // r.r
  __host__ __device__ int active() const { return 2; }
  __host__ __device__ int stopped() const { return 3; }
  __host__ __device__ int jused() const { return 4; }
  __host__ __device__ int nxt() const { return 5; }   // v_{j+1} is formed
  __host__ __device__ int nxh() const { return 6; }   // h_{j+1,j} (divisor of v_{j+1})
  __host__ __device__ int hn2() const { return 7; }   // w.w of the current step
  __host__ __device__ int H(int i, int j) const { return 8 + i * M + j; }  // (M+1) x M
  __host__ __device__ int cs(int i) const { return 8 + (M + 1) * M + i; }
  __host__ __device__ int sn(int i) const { return 8 + (M + 1) * M + M + i; }
  __host__ __device__ int gg(int i) const { return 8 + (M + 1) * M + 2 * M + i; }  // M + 1
  __host__ __device__ int y(int i) const { return 8 + (M + 1) * M + 3 * M + 1 + i; }
  __host__ __device__ int size() const { return 8 + (M + 1) * M + 4 * M + 1; }
};

// v0 = r / ||r|| when the pass is active (||r|| > rtol ||b||, krylov.py:63-70), else 0
__global__ void k_gm_start(const double* __restrict__ r, double* __restrict__ v0, double* __restrict__ g, GmLayout L,
                           long long n) {
  TMG_PDL_ENTRY;
  const double beta = sqrt(g[L.rr()]);
  const bool active = beta > GM_RTOL * sqrt(g[L.bb()]);
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v0[i] = active ? r[i] / beta : 0.0;
}
__global__ void k_gm_init(double* __restrict__ g, GmLayout L) {
  TMG_PDL_ENTRY;
  const double beta = sqrt(g[L.rr()]);
  const bool active = beta > GM_RTOL * sqrt(g[L.bb()]);
  for (int t = L.active(); t < L.size(); ++t) g[t] = 0.0;
  g[L.active()] = active ? 1.0 : 0.0;
  g[L.gg(0)] = beta;
}
// w -= g[k] * v   (MGS update with the Hessenberg entry just reduced into g[k])
__global__ void k_gm_axpy(double* __restrict__ w, const double* __restrict__ v, const double* __restrict__ g, int k,
                          long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) w[i] -= g[k] * v[i];
}
// step j bookkeeping: h_{j+1,j}, breakdown, previous rotations, new rotation,
// residual estimate and the stop test of krylov.py:104-121
__global__ void k_gm_rot(double* __restrict__ g, GmLayout L, int j) {
  TMG_PDL_ENTRY;
  g[L.nxt()] = 0.0;
  if (g[L.active()] == 0.0 || g[L.stopped()] != 0.0) return;
  const double tol = GM_RTOL * sqrt(g[L.bb()]);
  const double h = sqrt(g[L.hn2()]);
  g[L.H(j + 1, j)] = h;
  const bool bd = h < GM_BREAKDOWN;
  for (int i = 0; i < j; ++i) {
    const double c = g[L.cs(i)], s = g[L.sn(i)];
    const double t = c * g[L.H(i, j)] + s * g[L.H(i + 1, j)];
    g[L.H(i + 1, j)] = -s * g[L.H(i, j)] + c * g[L.H(i + 1, j)];
    g[L.H(i, j)] = t;
  }
  const double hjj = g[L.H(j, j)], hj1 = g[L.H(j + 1, j)];
  const double den = hypot(hjj, hj1);
  const double c = den != 0.0 ? hjj / den : 1.0, s = den != 0.0 ? hj1 / den : 0.0;
  g[L.cs(j)] = c;
  g[L.sn(j)] = s;
  g[L.H(j, j)] = den;
  g[L.H(j + 1, j)] = 0.0;
  g[L.gg(j + 1)] = -s * g[L.gg(j)];
  g[L.gg(j)] = c * g[L.gg(j)];
  g[L.jused()] = j + 1;
  const bool stop = fabs(g[L.gg(j + 1)]) <= tol || bd || j + 1 >= L.M;
  if (stop) g[L.stopped()] = 1.0;
  g[L.nxt()] = stop ? 0.0 : 1.0;
  g[L.nxh()] = h;
}
// v_{j+1} = w / h_{j+1,j} (zero once the cycle stopped)
__global__ void k_gm_next(const double* __restrict__ w, double* __restrict__ vn, const double* __restrict__ g,
                          GmLayout L, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) vn[i] = g[L.nxt()] != 0.0 ? w[i] / g[L.nxh()] : 0.0;
}
// y = triu(H[:j, :j])^-1 gg[:j]  (j = steps used), back substitution
__global__ void k_gm_solve(double* __restrict__ g, GmLayout L) {
  TMG_PDL_ENTRY;
  const int ju = (int)g[L.jused()];
  for (int i = 0; i < L.M; ++i) g[L.y(i)] = 0.0;
  if (g[L.active()] == 0.0) return;
  for (int i = ju - 1; i >= 0; --i) {
    double t = g[L.gg(i)];
    for (int k = i + 1; k < ju; ++k) t -= g[L.H(i, k)] * g[L.y(k)];
    g[L.y(i)] = t / g[L.H(i, i)];
  }
}
// x += Z y (the flexible correction, krylov.py:124-125); zero coefficients skip
// their basis vector
__global__ void k_gm_update(double* __restrict__ x, int x_zero, const double* __restrict__ Z, long long ldz,
                            const double* __restrict__ g, GmLayout L, long long n) {
  TMG_PDL_ENTRY;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (int j = 0; j < L.M; ++j) {
    const double yj = g[L.y(j)];
    if (yj != 0.0) d += yj * Z[j * ldz + i];
  }
  x[i] = (x_zero ? 0.0 : x[i]) + d;
}

// ----------------------------------------------------------------------------
// block Jacobi on a BSR level: inverses of the diagonal blocks (multigrid.py:64-95)
// ----------------------------------------------------------------------------
// Gauss-Jordan with partial pivoting per block row; bad |= 2 when |det| < 1e-300
template <int R>
__global__ void k_bsr_block_inv(BsrView<R, R> A, double* __restrict__ binv, unsigned* __restrict__ bad) {
  TMG_PDL_ENTRY;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  double m[R][R], inv[R][R];
#pragma unroll
  for (int a = 0; a < R; ++a)
#pragma unroll
    for (int b = 0; b < R; ++b) {
      m[a][b] = 0.0;
      inv[a][b] = a == b ? 1.0 : 0.0;
    }
  for (int p = A.rowptr[row]; p < A.rowptr[row + 1]; ++p)
    if (A.col[p] == row) {
#pragma unroll
      for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < R; ++b) m[a][b] = A.val[(long long)p * R * R + a * R + b];
    }
  double det = 1.0;
#pragma unroll
  for (int c = 0; c < R; ++c) {
    int piv = c;
#pragma unroll
    for (int a = c + 1; a < R; ++a)
      if (fabs(m[a][c]) > fabs(m[piv][c])) piv = a;
    if (piv != c) {
      det = -det;
#pragma unroll
      for (int b = 0; b < R; ++b) {
        double t = m[c][b]; m[c][b] = m[piv][b]; m[piv][b] = t;
        t = inv[c][b]; inv[c][b] = inv[piv][b]; inv[piv][b] = t;
      }
    }
    const double d = m[c][c];
    det *= d;
    const double rd = d != 0.0 ? 1.0 / d : 0.0;
#pragma unroll
    for (int b = 0; b < R; ++b) { m[c][b] *= rd; inv[c][b] *= rd; }
#pragma unroll
    for (int a = 0; a < R; ++a)
      if (a != c) {
        const double f = m[a][c];
#pragma unroll
        for (int b = 0; b < R; ++b) { m[a][b] -= f * m[c][b]; inv[a][b] -= f * inv[c][b]; }
      }
  }
  if (!(fabs(det) >= 1e-300)) atomicOr(bad, 2u);
#pragma unroll
  for (int a = 0; a < R; ++a)
#pragma unroll
    for (int b = 0; b < R; ++b) binv[((long long)row * R + a) * R + b] = inv[a][b];
}

// xo = x + w B^-1 (b - A x)   (x == nullptr: zero start, xo = w B^-1 b)
template <int R>
__global__ void __launch_bounds__(TPB) k_bsr_bjacobi(BsrView<R, R> A, const double* __restrict__ x,
                                                     const double* __restrict__ b, const double* __restrict__ binv,
                                                     const double* __restrict__ wp, double* __restrict__ xo) {
  TMG_PDL_ENTRY;
  int lane;
  const int row = bsr_row_id(A, lane);
  double out[R];
  if (x) {
    bsr_row<R, R>(A, row, lane, x, out);
  } else {
#pragma unroll
    for (int a = 0; a < R; ++a) out[a] = 0.0;
  }
  if (row >= A.nrows || lane != 0) return;
  const double w = *wp;
  double r[R];
#pragma unroll
  for (int a = 0; a < R; ++a) r[a] = b[(long long)row * R + a] - out[a];
#pragma unroll
  for (int a = 0; a < R; ++a) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < R; ++c) s += binv[((long long)row * R + a) * R + c] * r[c];
    const long long i = (long long)row * R + a;
    xo[i] = (x ? x[i] : 0.0) + w * s;
  }
}

}  // namespace tmg
