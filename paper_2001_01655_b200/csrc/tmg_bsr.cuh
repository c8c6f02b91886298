// Block-sparse (BSR) operators for the algebraic levels of the hierarchy:
// SA-AMG coarse operators (nvec x nvec blocks), prolongations P (bs x nvec) and
// restrictions P^T (nvec x bs).  Column indices are sorted within each block row
// (the reference's scipy CSR matrices are canonical, multigrid.py:262), blocks are
// row-major.  One thread per block row; the R outputs of a row stay in registers.
#pragma once
#include "tmg_ops.cuh"

namespace tmg {

struct Bsr {
  int nrows = 0, ncols = 0;  // block rows / block columns
  int R = 1, C = 1;          // block shape
  long long nnzb = 0;
  DevBuf<int> rowptr, col;
  DevBuf<double> val;
  long long scalar_nnz() const { return nnzb * R * C; }
};

template <int R, int C>
struct BsrView {
  const int* __restrict__ rowptr;
  const int* __restrict__ col;
  const double* __restrict__ val;
  int nrows;
};
template <int R, int C>
inline BsrView<R, C> view(const Bsr& m) {
  return BsrView<R, C>{m.rowptr.get(), m.col.get(), m.val.get(), m.nrows};
}

// y_row = sum_j A_rj x_j  (row of R outputs)
template <int R, int C>
__device__ __forceinline__ void bsr_row(const BsrView<R, C>& A, int row, const double* __restrict__ x,
                                        double out[R]) {
#pragma unroll
  for (int a = 0; a < R; ++a) out[a] = 0.0;
  const int e = A.rowptr[row + 1];
  for (int p = A.rowptr[row]; p < e; ++p) {
    const int j = A.col[p];
    double xv[C];
#pragma unroll
    for (int b = 0; b < C; ++b) xv[b] = __ldg(x + (long long)j * C + b);
    const double* blk = A.val + (long long)p * R * C;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < C; ++b) out[a] += __ldg(blk + a * C + b) * xv[b];
  }
}

// y = A x (+ y if accumulate)
template <int R, int C>
__global__ void __launch_bounds__(TPB) k_bsr_apply(BsrView<R, C> A, const double* __restrict__ x,
                                                   double* __restrict__ y, int accumulate) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  double out[R];
  bsr_row<R, C>(A, row, x, out);
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    y[i] = accumulate ? y[i] + out[a] : out[a];
  }
}

// bc = P^T r as a BSR product with the stored transpose; optional fused first
// zero-start Jacobi sweep of the coarse level, xc = w dinvc .* bc
template <int R, int C>
__global__ void __launch_bounds__(TPB) k_bsr_restrict(BsrView<R, C> Pt, const double* __restrict__ r,
                                                      double* __restrict__ bc, const double* __restrict__ dinvc,
                                                      const double* __restrict__ wp, double* __restrict__ xc) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= Pt.nrows) return;
  double out[R];
  bsr_row<R, C>(Pt, row, r, out);
  const double w = xc ? *wp : 0.0;
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    bc[i] = out[a];
    if (xc) xc[i] = w * dinvc[i] * out[a];
  }
}

// r = b - A x
template <int R>
__global__ void __launch_bounds__(TPB) k_bsr_residual(BsrView<R, R> A, const double* __restrict__ x,
                                                      const double* __restrict__ b, double* __restrict__ r) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  double out[R];
  bsr_row<R, R>(A, row, x, out);
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    r[i] = b[i] - out[a];
  }
}

// xo = x + w D^-1 (b - A x); DOT: reduce xo.b
template <int R, bool DOT>
__global__ void __launch_bounds__(TPB) k_bsr_jacobi(BsrView<R, R> A, const double* __restrict__ x,
                                                    const double* __restrict__ b, const double* __restrict__ dinv,
                                                    const double* __restrict__ wp, double* __restrict__ xo, Red red) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (row < A.nrows) {
    const double w = *wp;
    double out[R];
    bsr_row<R, R>(A, row, x, out);
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const long long i = (long long)row * R + a;
      const double xn = x[i] + w * (dinv[i] * (b[i] - out[a]));
      xo[i] = xn;
      if (DOT) v += xn * b[i];
    }
  }
  if (DOT) grid_reduce(v, red);
}

// One Chebyshev step on a BSR level: p' = D^-1 r + beta p; x += alpha p'; r' = r - alpha A p'
// (p' of neighbours is needed, so p' is produced by k_bsr_cheb_p first).
__global__ void k_bsr_cheb_p(const double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ dinv, const double* __restrict__ coef, int step,
                             double* __restrict__ po, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double beta = step == 0 ? 0.0 : coef[2 * step + 1];
  const double z = dinv[i] * r[i];
  po[i] = beta == 0.0 ? z : z + beta * p[i];
}
template <int R>
__global__ void __launch_bounds__(TPB) k_bsr_cheb(BsrView<R, R> A, const double* __restrict__ r,
                                                  const double* __restrict__ pn, const double* __restrict__ coef,
                                                  int step, int x_zero, double* __restrict__ x,
                                                  double* __restrict__ ro) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  const double alpha = coef[2 * step];
  double out[R];
  bsr_row<R, R>(A, row, pn, out);
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    x[i] = (x_zero ? 0.0 : x[i]) + alpha * pn[i];
    ro[i] = r[i] - alpha * out[a];
  }
}

// y = ds .* A (ds .* v)
template <int R>
__global__ void __launch_bounds__(TPB) k_bsr_apply_sym(BsrView<R, R> A, const double* __restrict__ v,
                                                       const double* __restrict__ ds, double* __restrict__ tmp,
                                                       double* __restrict__ y) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  double out[R];
  bsr_row<R, R>(A, row, tmp, out);
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const long long i = (long long)row * R + a;
    y[i] = ds[i] * out[a];
  }
}
__global__ void k_vmul(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ y, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) y[i] = a[i] * b[i];
}

// scalar diagonal of a square BSR
template <int R>
__global__ void k_bsr_diag(BsrView<R, R> A, double* __restrict__ d, unsigned* __restrict__ bad) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  double dv[R];
#pragma unroll
  for (int a = 0; a < R; ++a) dv[a] = 0.0;
  for (int p = A.rowptr[row]; p < A.rowptr[row + 1]; ++p)
    if (A.col[p] == row) {
#pragma unroll
      for (int a = 0; a < R; ++a) dv[a] = A.val[(long long)p * R * R + a * R + a];
    }
#pragma unroll
  for (int a = 0; a < R; ++a) {
    d[(long long)row * R + a] = dv[a];
    if (dv[a] == 0.0) atomicOr(bad, 1u);
  }
}

// dense row-major copy of a square BSR (coarsest level)
template <int R>
__global__ void k_bsr_to_dense(BsrView<R, R> A, double* __restrict__ Ad, long long n) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= A.nrows) return;
  for (int p = A.rowptr[row]; p < A.rowptr[row + 1]; ++p) {
    const int j = A.col[p];
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b)
        Ad[((long long)row * R + a) * n + (long long)j * R + b] = A.val[(long long)p * R * R + a * R + b];
  }
}

// Dispatch helpers over the block shapes used by SA-AMG (dpn in {2,3}, nvec in {3,6}).
#define TMG_BSR_SQUARE_DISPATCH(Rv, ...)                        \
  switch (Rv) {                                                 \
    case 1: { constexpr int RR = 1; __VA_ARGS__; } break;        \
    case 2: { constexpr int RR = 2; __VA_ARGS__; } break;        \
    case 3: { constexpr int RR = 3; __VA_ARGS__; } break;        \
    case 6: { constexpr int RR = 6; __VA_ARGS__; } break;        \
    default: throw Error(-1, "unsupported BSR block size");     \
  }
#define TMG_BSR_RECT_DISPATCH(Rv, Cv, ...)                                              \
  if (Rv == 2 && Cv == 3) { constexpr int RR = 2, CC = 3; __VA_ARGS__; }                \
  else if (Rv == 3 && Cv == 2) { constexpr int RR = 3, CC = 2; __VA_ARGS__; }           \
  else if (Rv == 3 && Cv == 6) { constexpr int RR = 3, CC = 6; __VA_ARGS__; }           \
  else if (Rv == 6 && Cv == 3) { constexpr int RR = 6, CC = 3; __VA_ARGS__; }           \
  else if (Rv == 3 && Cv == 3) { constexpr int RR = 3, CC = 3; __VA_ARGS__; }           \
  else if (Rv == 6 && Cv == 6) { constexpr int RR = 6, CC = 6; __VA_ARGS__; }           \
  else if (Rv == 2 && Cv == 2) { constexpr int RR = 2, CC = 2; __VA_ARGS__; }           \
  else if (Rv == 1 && Cv == 3) { constexpr int RR = 1, CC = 3; __VA_ARGS__; }           \
  else if (Rv == 3 && Cv == 1) { constexpr int RR = 3, CC = 1; __VA_ARGS__; }           \
  else if (Rv == 1 && Cv == 6) { constexpr int RR = 1, CC = 6; __VA_ARGS__; }           \
  else if (Rv == 6 && Cv == 1) { constexpr int RR = 6, CC = 1; __VA_ARGS__; }           \
  else if (Rv == 1 && Cv == 1) { constexpr int RR = 1, CC = 1; __VA_ARGS__; }           \
  else throw Error(-1, "unsupported BSR block shape");

}  // namespace tmg
